set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/r2am_pytest.txt 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2am_pytest.txt
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_kernels.py --only attn > gpurun_out/r2am_san_attn_$tool.txt 2>&1; echo "san attn $tool rc=$?"; grep -E "SUMMARY" gpurun_out/r2am_san_attn_$tool.txt | tail -1
  ASKV_ATTN_PAIR=1 timeout 900 compute-sanitizer --tool $tool python tools/sanitize_kernels.py --only batch > gpurun_out/r2am_san_batch_$tool.txt 2>&1; echo "san batch $tool rc=$?"; grep -E "SUMMARY" gpurun_out/r2am_san_batch_$tool.txt | tail -1
done
timeout 900 python bench.py > gpurun_out/r2am_bench.log 2>&1; echo "bench rc=$?"
