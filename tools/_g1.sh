set -x
(free -g; nproc; lscpu | head -20; nvidia-smi topo -m; numactl -H 2>&1 | head; df -h /tmp /root; cat /sys/devices/system/node/online; ls /sys/devices/system/node) > gpurun_out/boxinfo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
for t in racecheck synccheck initcheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/san_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/san_rc.txt
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/san_rc.txt
