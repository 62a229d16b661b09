# A/B: warp-converged MMA issue with the lane elected inside the asm (1) vs `if (lane == 0)` (0); parity tests of (1).
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -DASKV_ATTN_ELECT_ISSUE=0 -o /tmp/avt_e0 > gpurun_out/r3t_b0.txt 2>&1 &
$B -o /tmp/avt_e1 > gpurun_out/r3t_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in e0 e1; do timeout 60 /tmp/avt_$v > gpurun_out/r3t_avt_${v}_$i.txt 2>&1; done; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py tests/test_rope_api_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3t_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3t_rc.txt
