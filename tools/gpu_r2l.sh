set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
CLTK_TRACE=1 timeout 300 python tools/e2e_trace.py > $O/e2e_trace.txt 2>&1
