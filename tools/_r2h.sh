set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/r2h_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h_rc.txt
timeout 300 python tools/kbench.py attn --reps 20 --warm --batch 20 > gpurun_out/r2h_kb_sk.txt 2>&1
timeout 300 python tools/kbench.py attn --reps 20 > gpurun_out/r2h_kb_sk_cold.txt 2>&1
ASKV_ATTN_SK=0 timeout 300 python tools/kbench.py attn --reps 20 > gpurun_out/r2h_kb_old_cold.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_ncu_times.csv python tools/kbench.py attn --shape 2142,237,40,40 --reps 2 > /dev/null 2>&1
