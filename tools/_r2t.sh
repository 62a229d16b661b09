set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/host_batch.py > gpurun_out/r2t_host_batch.txt 2>&1
timeout 600 python tools/host_batch.py --no-batch > gpurun_out/r2t_host_nobatch.txt 2>&1
