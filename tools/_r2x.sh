set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2x_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2x_rc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2x_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2x_rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_ab.cu -o /tmp/ab -lcuda && /tmp/ab tma > gpurun_out/r2x_ab.txt 2>&1 && /tmp/ab tma >> gpurun_out/r2x_ab.txt 2>&1
timeout 900 python bench.py --serve-dram-gb 0 > gpurun_out/r2x_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2x_rc.txt
