# round-2 first GPU pass: tests, smoke, sanitizers on the K2/K3 kernels, a bench line
set -x
mkdir -p gpurun_out
(nvidia-smi; nvidia-smi topo -m; lscpu | head -25; numactl -H 2>&1 | head -20; free -g) > gpurun_out/r2a_boxinfo.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_rc.txt
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_kernels.py --only attn > gpurun_out/r2a_san_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/r2a_rc.txt
done
for t in initcheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/r2a_san_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/r2a_rc.txt
done
timeout 900 python bench.py > gpurun_out/r2a_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2a_rc.txt
