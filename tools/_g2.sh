for t in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_kernels.py --only attn > gpurun_out/san2_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/san2_rc.txt
done
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_kernels.py --only provenance > gpurun_out/san2_initcheck_prov.txt 2>&1; echo "initprov rc=$?" >> gpurun_out/san2_rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/san2_rc.txt
