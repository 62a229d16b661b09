set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_batch.csv python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/r2s_l1.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 82 -c 1 -o gpurun_out/r2s_attn_full python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/r2s_l2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reembed -s 1300 -c 1 -o gpurun_out/r2s_reembed_full python tools/step_profile.py --mode hbm --turns 16 --batch --no-profiler > gpurun_out/r2s_l3.txt 2>&1
timeout 600 python tools/step_profile.py --mode hbm --turns 16 --batch > gpurun_out/r2s_step_batch.json 2> gpurun_out/r2s_step_batch.err
timeout 600 python tools/step_profile.py --mode hbm --turns 16 > gpurun_out/r2s_step_unbatched.json 2> gpurun_out/r2s_step_unbatched.err
