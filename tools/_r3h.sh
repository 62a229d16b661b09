# Same-box A/B: V slot released right after PV_B(j) (early) vs after S_B(j+1); kernel parity tests.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -DASKV_ATTN_EARLY_VFREE=0 -o /tmp/avt_v0 > gpurun_out/r3h_b0.txt 2>&1 &
$B -o /tmp/avt_v1 > gpurun_out/r3h_b1.txt 2>&1 &
$B -DASKV_ATTN_PROBE=1 -o /tmp/avt_v1p1 > gpurun_out/r3h_b2.txt 2>&1 &
wait
for i in 1 2 3; do for v in v0 v1; do timeout 120 /tmp/avt_$v > gpurun_out/r3h_avt_${v}_$i.txt 2>&1; done; done
timeout 120 /tmp/avt_v1p1 > gpurun_out/r3h_avt_v1p1_1.txt 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py -m gpu -x -q --timeout 200 > gpurun_out/r3h_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3h_rc.txt
