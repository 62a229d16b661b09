nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_sk_trace.cu -o /tmp/attn_sk_trace -lcuda
mkdir -p gpurun_out
ASKV_ATTN_SK=1 /tmp/attn_sk_trace 2142 237 40 > gpurun_out/r2n_trace.txt 2>&1
