set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/r2m_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m_rc.txt
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude"
$B tools/attn_ab.cu -o /tmp/ab -lcuda
/tmp/ab grid > gpurun_out/r2m_ab.txt 2>&1
ASKV_ATTN_SK=1 /tmp/ab sk >> gpurun_out/r2m_ab.txt 2>&1
/tmp/ab grid >> gpurun_out/r2m_ab.txt 2>&1
ASKV_ATTN_SK=1 /tmp/ab sk >> gpurun_out/r2m_ab.txt 2>&1
$B -DASKV_ATTN_TRACE tools/attn_sk_trace.cu -o /tmp/attn_sk_trace -lcuda
ASKV_ATTN_SK=1 /tmp/attn_sk_trace 2142 237 40 > gpurun_out/r2m_trace.txt 2>&1
