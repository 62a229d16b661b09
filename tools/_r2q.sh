set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2q_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2q_rc.txt
timeout 400 python -X faulthandler -c "
import faulthandler, sys
faulthandler.dump_traceback_later(300, exit=True)
import pytest
sys.exit(pytest.main(['tests/test_batch_gpu.py', '-q']))
" > gpurun_out/r2q_batch.txt 2>&1; echo "batch rc=$?" >> gpurun_out/r2q_rc.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2q_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2q_rc.txt
timeout 900 python bench.py --serve-dram-gb 0 > gpurun_out/r2q_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r2q_rc.txt
