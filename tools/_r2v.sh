set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2v_rc.txt
timeout 600 python tools/host_batch.py > gpurun_out/r2v_host_batch.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2v_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2v_rc.txt
timeout 900 python bench.py --serve-dram-gb 0 > gpurun_out/r2v_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2v_rc.txt
