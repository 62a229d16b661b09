# Round-2 closing sweep (rh_: descriptor-base MMA issue, per-warp P arrival) on the committed code: build, smoke, GPU tests,
# sanitizers on the batched pass, benches (C3 default + reference arm, C2, C4,
# C5 rank probe), launch list and full ncu captures of the batched step.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rh_build.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rh_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/rh_rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/rh_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/rh_rc.txt
for tool in racecheck synccheck memcheck; do
  ASKV_ATTN_PAIR=1 timeout 900 compute-sanitizer --tool $tool python tools/sanitize_kernels.py --only batch > gpurun_out/rh_san_batch_$tool.txt 2>&1; echo "san $tool rc=$?" >> gpurun_out/rh_rc.txt
done
timeout 900 python bench.py > gpurun_out/rh_bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/rh_rc.txt
timeout 600 python bench.py --impl reference > gpurun_out/rh_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/rh_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rh_launches_batch.csv python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/rh_l1.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 82 -c 1 -o gpurun_out/rh_attn_full python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/rh_l2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reembed -s 90 -c 1 -o gpurun_out/rh_reembed_full python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/rh_l3.txt 2>&1
timeout 600 python tools/step_profile.py --mode hbm --turns 16 --batch > gpurun_out/rh_step_batch.json 2> gpurun_out/rh_step_batch.err
for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/rh_bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/rh_rc.txt; done
