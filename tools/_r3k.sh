# Final code: smoke, full GPU tests, C3 bench + reference arm, launch list of the batched step.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3k_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r3k_rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r3k_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r3k_rc.txt
timeout 900 python bench.py > gpurun_out/r3k_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r3k_rc.txt
timeout 600 python bench.py --impl reference > gpurun_out/r3k_bench_ref.txt 2>&1; echo "ref rc=$?" >> gpurun_out/r3k_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3k_launches_batch.csv python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/r3k_l1.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 82 -c 1 -o gpurun_out/r3k_attn_full python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/r3k_l2.txt 2>&1
