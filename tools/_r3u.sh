# Exact final tree: smoke, full GPU tests, C3 bench.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3u_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r3u_rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r3u_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3u_rc.txt
timeout 900 python bench.py > gpurun_out/r3u_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r3u_rc.txt
