# A/B: one tcgen05 fence after the ring + P waits of a paired iteration (1) vs a fence after each wait (0); parity of (1).
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -DASKV_ATTN_ONE_FENCE=0 -o /tmp/avt_f0 > gpurun_out/r3v_b0.txt 2>&1 &
$B -o /tmp/avt_f1 > gpurun_out/r3v_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in f0 f1; do timeout 60 /tmp/avt_$v > gpurun_out/r3v_avt_${v}_$i.txt 2>&1; done; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py tests/test_rope_api_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3v_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3v_rc.txt
