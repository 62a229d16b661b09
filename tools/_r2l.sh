set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_trace.cu -o /tmp/attn_trace -lcuda
/tmp/attn_trace 2142 237 40 > gpurun_out/r2l_trace.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 compute-sanitizer --tool initcheck --print-limit 10 python tools/sanitize_kernels.py --only provenance > gpurun_out/r2l_init_prov.txt 2>&1
