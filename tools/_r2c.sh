set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/link_probe tools/link_probe.cu && timeout 300 /tmp/link_probe > gpurun_out/r2c_link.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_measured_gpu.py tests/test_rope_api_gpu.py -x -q > gpurun_out/r2c_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_rc.txt
timeout 300 python tools/kbench.py attn --reps 30 > gpurun_out/r2c_kbench_sk.txt 2>&1
ASKV_ATTN_SK=0 timeout 300 python tools/kbench.py attn --reps 30 > gpurun_out/r2c_kbench_nosk.txt 2>&1
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_kernels.py --only attn > gpurun_out/r2c_san_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/r2c_rc.txt
done
timeout 1500 python -m paper_2403_19708_b200.serve --config c3 --shard 0 --of 8 --turns-out --json gpurun_out/r2c_serve_c3_s0of8.json > gpurun_out/r2c_serve.txt 2>&1; echo "serve rc=$?" >> gpurun_out/r2c_rc.txt
