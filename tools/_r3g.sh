# K3 pipeline probes (varlen launch): full kernel vs no softmax work (p1) vs S loads only (p2);
# plus the HBM-tier eviction test with its new oracle assertions.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -o /tmp/avt_full > gpurun_out/r3g_b0.txt 2>&1 &
$B -DASKV_ATTN_PROBE=1 -o /tmp/avt_p1 > gpurun_out/r3g_b1.txt 2>&1 &
$B -DASKV_ATTN_PROBE=2 -o /tmp/avt_p2 > gpurun_out/r3g_b2.txt 2>&1 &
wait
for i in 1 2; do for v in full p1 p2; do timeout 120 /tmp/avt_$v > gpurun_out/r3g_avt_${v}_$i.txt 2>&1; done; done
timeout 600 python -m pytest tests/test_engine_gpu.py -m gpu -q --timeout 300 -k "hbm_tier" > gpurun_out/r3g_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3g_rc.txt
