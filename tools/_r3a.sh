# Session re-entry check of HEAD: build, smoke, GPU tests, C3 bench, varlen K3 baseline.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3a_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r3a_rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_varlen_trace.cu -o /tmp/avt -lcuda > gpurun_out/r3a_avt_build.txt 2>&1
for i in 1 2; do timeout 120 /tmp/avt > gpurun_out/r3a_avt_$i.txt 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r3a_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3a_rc.txt
timeout 900 python bench.py > gpurun_out/r3a_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r3a_rc.txt
