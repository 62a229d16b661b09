mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sanitize_kernels.py --only batch > gpurun_out/r2ab_batch.txt 2>&1; echo "plain rc=$?" >> gpurun_out/r2ab_rc.txt
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_kernels.py --only batch > gpurun_out/r2ab_san_batch_$t.txt 2>&1; echo "batch $t rc=$?" >> gpurun_out/r2ab_rc.txt
done
timeout 900 python -m pytest tests/test_batch_gpu.py -q --timeout 300 > gpurun_out/r2ab_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ab_rc.txt
