set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.txt 2>&1
timeout 900 python -m pytest tests/test_measured_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/r2b_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_rc.txt
timeout 1200 python -m paper_2403_19708_b200.serve --config c3 --shard 0 --of 8 --turns-out --json gpurun_out/r2b_serve_c3_s0of8.json > gpurun_out/r2b_serve.txt 2>&1; echo "serve rc=$?" >> gpurun_out/r2b_rc.txt
ASKV_COPY_2D=0 timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2b_bench_no2d.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2b_rc.txt
