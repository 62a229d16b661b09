# K3 probe 4 (no softmax, no K/V copies, no ring waits after the first fill) vs probe 3.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -DASKV_ATTN_PROBE=3 -o /tmp/avt_p3 > gpurun_out/r3q_b3.txt 2>&1 &
$B -DASKV_ATTN_PROBE=4 -o /tmp/avt_p4 > gpurun_out/r3q_b4.txt 2>&1 &
wait
for i in 1 2; do for v in p3 p4; do timeout 60 /tmp/avt_$v > gpurun_out/r3q_avt_${v}_$i.txt 2>&1; done; done
