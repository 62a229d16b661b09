set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2i_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2i_rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i_rc.txt
timeout 300 python tools/kbench.py reembed > gpurun_out/r2i_kb_reembed.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r2i_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2i_rc.txt
