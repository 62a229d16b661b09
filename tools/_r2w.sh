set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python bench.py > gpurun_out/r2w_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2w_rc.txt
timeout 900 python bench.py --impl reference > gpurun_out/r2w_ref.txt 2>&1; echo "ref rc=$?" >> gpurun_out/r2w_rc.txt
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2w_c2.txt 2>&1; echo "c2 rc=$?" >> gpurun_out/r2w_rc.txt
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2w_c4.txt 2>&1; echo "c4 rc=$?" >> gpurun_out/r2w_rc.txt
timeout 900 python bench.py --config c5 --tp-rank-of 8 --no-cpu-baseline > gpurun_out/r2w_c5.txt 2>&1; echo "c5 rc=$?" >> gpurun_out/r2w_rc.txt
ASKV_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --turns 4 --steps 2 --warmup 3 --serve-dram-gb 0 --no-cpu-baseline > gpurun_out/r2w_n2.txt 2>&1; echo "n2 rc=$?" >> gpurun_out/r2w_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2w_launches_unbatched.csv python tools/step_profile.py --mode hbm --turns 16 --no-profiler > /dev/null 2>&1
