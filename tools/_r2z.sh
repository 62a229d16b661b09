set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2z_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z_rc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2z_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2z_rc.txt
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_kernels.py --only batch > gpurun_out/r2z_san_batch_$t.txt 2>&1; echo "batch $t rc=$?" >> gpurun_out/r2z_rc.txt
done
timeout 900 python bench.py --serve-dram-gb 0 > gpurun_out/r2z_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2z_rc.txt
