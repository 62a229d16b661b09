set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.txt 2>&1
for c in 40 80 120 148; do
echo "ctas=$c" >> gpurun_out/r2e_kb.txt
ASKV_ATTN_SK_CTAS=$c timeout 300 python tools/kbench.py attn --shape 2142,237,40,40 --reps 20 --warm --batch 20 >> gpurun_out/r2e_kb.txt 2>&1
done
ASKV_ATTN_SK=0 timeout 300 python tools/kbench.py attn --shape 2142,237,40,40 --reps 20 --warm --batch 20 >> gpurun_out/r2e_kb.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_ncu_times.csv python tools/kbench.py attn --shape 2142,237,40,40 --reps 2 > /dev/null 2>&1
ASKV_ATTN_SK=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_ncu_times_old.csv python tools/kbench.py attn --shape 2142,237,40,40 --reps 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_sk_kernel -c 1 -o gpurun_out/r2e_sk_full python tools/kbench.py attn --shape 2142,237,40,40 --reps 1 > gpurun_out/r2e_ncu_full.log 2>&1
