set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_sk_trace.cu -o /tmp/attn_sk_trace -lcuda > gpurun_out/r2f_build.txt 2>&1
/tmp/attn_sk_trace 2142 237 40 > gpurun_out/r2f_trace.txt 2>&1
ASKV_ATTN_SK_CTAS=80 /tmp/attn_sk_trace 2142 237 40 >> gpurun_out/r2f_trace.txt 2>&1
