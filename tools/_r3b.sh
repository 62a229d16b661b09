# Column-split softmax (K3 paired instance): parity + isolated varlen-launch A/B.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_varlen_trace.cu -lcuda"
$B -o /tmp/avt1 > gpurun_out/r3b_avt_build1.txt 2>&1 &
$B -DASKV_ATTN_COLSPLIT=0 -o /tmp/avt0 > gpurun_out/r3b_avt_build0.txt 2>&1 &
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3b_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3b_rc.txt
wait
for i in 1 2; do timeout 120 /tmp/avt1 > gpurun_out/r3b_avt1_$i.txt 2>&1; echo "avt1 rc=$?" >> gpurun_out/r3b_rc.txt; timeout 120 /tmp/avt0 > gpurun_out/r3b_avt0_$i.txt 2>&1; done
