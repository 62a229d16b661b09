# Same-box A/B of the varlen K3 launch: HEAD kernel vs descriptor-base MMA issue
# (column split off / on, on with 3/8 polynomial exps); then the C3 bench.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda"
$B tools/_avt_head.cu -o /tmp/avt_head > gpurun_out/r3c_b0.txt 2>&1 &
$B tools/attn_varlen_trace.cu -o /tmp/avt_new > gpurun_out/r3c_b1.txt 2>&1 &
$B -DASKV_ATTN_COLSPLIT=1 tools/attn_varlen_trace.cu -o /tmp/avt_col > gpurun_out/r3c_b2.txt 2>&1 &
$B -DASKV_ATTN_COLSPLIT=1 -DASKV_ATTN_POLY_Q=2 tools/attn_varlen_trace.cu -o /tmp/avt_colp2 > gpurun_out/r3c_b3.txt 2>&1 &
wait
for i in 1 2 3; do for v in head new col colp2; do timeout 120 /tmp/avt_$v > gpurun_out/r3c_avt_${v}_$i.txt 2>&1; done; done
timeout 900 python bench.py > gpurun_out/r3c_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r3c_rc.txt
