# GPU suite after the host-model restatement; where the C4 batch e2e call spends its host time
set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_x.log 2>&1; echo "pytest rc=$?" >> $O/pytest_x.log
CLTK_TRACE=1 timeout 300 python bench.py --workload worst_off_batch --paths-per-gpu 2000000 --no-cpu-baseline --e2e-steps 4 > $O/x_wob.json 2> $O/x_wob.err
grep cltk $O/x_wob.err | tail -8 > $O/x_wob_trace.txt
echo done
