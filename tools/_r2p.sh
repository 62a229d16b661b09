set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2p_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2p_rc.txt
timeout 900 python -m pytest tests/test_batch_gpu.py -x -q > gpurun_out/r2p_batch.txt 2>&1; echo "batch rc=$?" >> gpurun_out/r2p_rc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2p_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_rc.txt
timeout 1800 python bench.py --serve-dram-gb 0 > gpurun_out/r2p_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2p_rc.txt
