# A/B: S_A(j+1) interleaved with PV_B(j) (1) vs sequential (0); parity of the interleaved build.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -o /tmp/avt_i0 > gpurun_out/r3p_b0.txt 2>&1 &
$B -DASKV_ATTN_INTERLEAVE=1 -o /tmp/avt_i1 > gpurun_out/r3p_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in i0 i1; do timeout 120 /tmp/avt_$v > gpurun_out/r3p_avt_${v}_$i.txt 2>&1; done; done
