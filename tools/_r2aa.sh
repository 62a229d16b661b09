mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sanitize_kernels.py --only batch > gpurun_out/r2aa_batch.txt 2>&1
ASKV_VARLEN=0 python tools/sanitize_kernels.py --only batch >> gpurun_out/r2aa_batch.txt 2>&1
