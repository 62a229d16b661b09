# K/V L2 policy A/B (evict_last vs evict_first) on the varlen launch; then the final code's
# smoke, full GPU tests and C3 bench.
set -x
mkdir -p gpurun_out
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude -lcuda tools/attn_varlen_trace.cu"
$B -o /tmp/avt_pl1 > gpurun_out/r3i_b1.txt 2>&1 &
$B -DASKV_ATTN_KV_POLICY=2 -o /tmp/avt_pl2 > gpurun_out/r3i_b2.txt 2>&1 &
wait
for i in 1 2 3; do for v in pl1 pl2; do timeout 120 /tmp/avt_$v > gpurun_out/r3i_avt_${v}_$i.txt 2>&1; done; done
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3i_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r3i_rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r3i_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3i_rc.txt
timeout 900 python bench.py > gpurun_out/r3i_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r3i_rc.txt
