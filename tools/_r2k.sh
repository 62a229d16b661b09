set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude"
$B tools/attn_ab.cu -o /tmp/ab_base -lcuda &
$B -DASKV_MBAR_SUSPEND_NS=10000000 tools/attn_ab.cu -o /tmp/ab_susp -lcuda &
$B -DASKV_ATTN_POLY_Q=2 tools/attn_ab.cu -o /tmp/ab_poly2 -lcuda &
$B -DASKV_ATTN_POLY_Q=0 tools/attn_ab.cu -o /tmp/ab_poly0 -lcuda &
$B -DASKV_ATTN_TRACE tools/attn_trace.cu -o /tmp/attn_trace -lcuda &
wait
for r in 1 2; do for v in base susp poly2 poly0; do /tmp/ab_$v $v >> gpurun_out/r2k_ab.txt 2>&1; done; done
/tmp/attn_trace 2142 237 40 > gpurun_out/r2k_trace.txt 2>&1
