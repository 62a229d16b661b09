set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.txt 2>&1
for sk in 1 0; do
ASKV_ATTN_SK=$sk timeout 300 python tools/kbench.py attn --shape 2142,237,40,40 --reps 20 --warm --batch 20 >> gpurun_out/r2d_kb.txt 2>&1
ASKV_ATTN_SK=$sk timeout 300 python tools/kbench.py attn --shape 1000,100,40,40 --reps 20 --warm --batch 20 >> gpurun_out/r2d_kb.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_ncu_sk.csv python tools/kbench.py attn --shape 2142,237,40,40 --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "nccl or tensor_parallel" > gpurun_out/r2d_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_rc.txt
