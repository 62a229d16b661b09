# Does a long run slow the tensor core per clock?  mma_probe2's K3 MMA sequence at 400 vs 40000 iterations (grid 148).
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude tools/mma_probe2.cu -o /tmp/mp2 -lcuda > gpurun_out/r3r_b.txt 2>&1
for it in 400 4000 40000; do MIX_ONLY=1 ITERS=$it timeout 120 /tmp/mp2 > gpurun_out/r3r_mp2_$it.txt 2>&1; done
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv > gpurun_out/r3r_smi.txt 2>&1
