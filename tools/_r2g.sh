set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/r2g_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_rc.txt
timeout 300 python tools/kbench.py attn --reps 20 --warm --batch 20 > gpurun_out/r2g_kb_sk.txt 2>&1
ASKV_ATTN_SK=0 timeout 300 python tools/kbench.py attn --reps 20 --warm --batch 20 > gpurun_out/r2g_kb_old.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_sk_trace.cu -o /tmp/attn_sk_trace -lcuda > gpurun_out/r2g_tbuild.txt 2>&1
/tmp/attn_sk_trace 2142 237 40 > gpurun_out/r2g_trace.txt 2>&1
