A="--no-cpu-baseline --disk-dir none --decode-steps 0"
ASKV_BENCH_CLOCKS=0 timeout 900 python bench.py $A > gpurun_out/bench_noclk.json 2> gpurun_out/bench_noclk.err
timeout 900 python bench.py $A > gpurun_out/bench_clk.json 2> gpurun_out/bench_clk.err
