# Re-tune after the o_full change (same box): ring split K3/V2 (default) vs K2/V3; 1/4 (default) vs 0 / 3/8 (mask 0x8A) polynomial exps.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -o /tmp/avt_base > gpurun_out/r3l_b0.txt 2>&1 &
$B -DASKV_ATTN_PAIR_KSTAGES=2 -DASKV_ATTN_PAIR_VSTAGES=3 -o /tmp/avt_k2v3 > gpurun_out/r3l_b1.txt 2>&1 &
$B -DASKV_ATTN_POLY_Q=0 -o /tmp/avt_poly0 > gpurun_out/r3l_b2.txt 2>&1 &
$B -DASKV_ATTN_POLY_MASK=0x8A -o /tmp/avt_poly38 > gpurun_out/r3l_b3.txt 2>&1 &
wait
for i in 1 2 3; do for v in base k2v3 poly0 poly38; do timeout 120 /tmp/avt_$v > gpurun_out/r3l_avt_${v}_$i.txt 2>&1; done; done
