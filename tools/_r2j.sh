set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2j_rc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2j_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2j_rc.txt
for m in provenance engine_graph engine_stream; do
  timeout 600 compute-sanitizer --tool initcheck --print-limit 30 python tools/sanitize_kernels.py --only $m > gpurun_out/r2j_init_$m.txt 2>&1; echo "init $m rc=$?" >> gpurun_out/r2j_rc.txt
done
ASKV_ATTN_SK=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_kernels.py --only attn > gpurun_out/r2j_san_sk_racecheck.txt 2>&1; echo "sk racecheck rc=$?" >> gpurun_out/r2j_rc.txt
ASKV_ATTN_SK=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_kernels.py --only attn > gpurun_out/r2j_san_sk_synccheck.txt 2>&1; echo "sk synccheck rc=$?" >> gpurun_out/r2j_rc.txt
timeout 1800 python bench.py > gpurun_out/r2j_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2j_rc.txt
