# Same-box A/B: P-ready barrier with one arrival per softmax warp (1) vs per thread (0).
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -DASKV_ATTN_WARP_ARRIVE=0 -o /tmp/avt_wa0 > gpurun_out/r3e_b0.txt 2>&1 &
$B -o /tmp/avt_wa1 > gpurun_out/r3e_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in wa0 wa1; do timeout 120 /tmp/avt_$v > gpurun_out/r3e_avt_${v}_$i.txt 2>&1; done; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3e_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3e_rc.txt
