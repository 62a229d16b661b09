# mma_probe2 MIX sequence with the probe's own shared-memory map (KMAP=0) vs K3's paired map (KMAP=1); KMAP=2 adds the kernel's wait + tcgen05 fence before each group.
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2403_19708_b200/csrc -Iinclude tools/mma_probe2.cu -o /tmp/mp2 -lcuda > gpurun_out/r3s_b.txt 2>&1
for m in 0 2; do MIX_ONLY=1 KMAP=$m ITERS=4000 timeout 120 /tmp/mp2 > gpurun_out/r3s_mp2_kmap$m.txt 2>&1; done
