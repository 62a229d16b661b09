set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 compute-sanitizer --tool initcheck --print-limit 10 python tools/sanitize_kernels.py --only provenance > gpurun_out/r2o_init_prov.txt 2>&1
free -g > gpurun_out/r2o_free.txt
timeout 2400 python -m paper_2403_19708_b200.serve --config c3 --of 1 --dram-gb 112 --hbm-gb 64 --turns-out --json gpurun_out/r2o_serve_c3_full.json > gpurun_out/r2o_serve.txt 2>&1; echo "serve rc=$?" >> gpurun_out/r2o_rc.txt
