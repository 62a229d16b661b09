# Unpaired instance: o_full by the last PV only (ALL=1) vs every PV, single-launch shapes (tools/attn_ab.cu).
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_ab.cu -lcuda"
$B -o /tmp/ab_0 > gpurun_out/r3m_b0.txt 2>&1 &
$B -DASKV_ATTN_LAST_OFULL_ALL=1 -o /tmp/ab_1 > gpurun_out/r3m_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in 0 1; do timeout 120 /tmp/ab_$v ofull_all=$v >> gpurun_out/r3m_ab.txt 2>&1; done; done
