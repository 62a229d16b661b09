# Same-box A/B: K(j+1) waited at its first S (new) vs before PV_A(j) (head); kernel parity tests.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda"
$B tools/_avt_head.cu -o /tmp/avt_head > gpurun_out/r3d_b0.txt 2>&1 &
$B tools/attn_varlen_trace.cu -o /tmp/avt_new > gpurun_out/r3d_b1.txt 2>&1 &
wait
for i in 1 2 3; do for v in head new; do timeout 120 /tmp/avt_$v > gpurun_out/r3d_avt_${v}_$i.txt 2>&1; done; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3d_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3d_rc.txt
