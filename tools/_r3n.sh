# K3 pipeline probes on the final kernel: full / no softmax (p1) / no softmax and no K/V copies after the first ring fill (p3).
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -o /tmp/avt_full > gpurun_out/r3n_b0.txt 2>&1 &
$B -DASKV_ATTN_PROBE=1 -o /tmp/avt_p1 > gpurun_out/r3n_b1.txt 2>&1 &
$B -DASKV_ATTN_PROBE=3 -o /tmp/avt_p3 > gpurun_out/r3n_b3.txt 2>&1 &
wait
for i in 1 2; do for v in full p1 p3; do timeout 120 /tmp/avt_$v > gpurun_out/r3n_avt_${v}_$i.txt 2>&1; done; done
