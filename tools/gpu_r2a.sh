#!/bin/bash
# Round-2 session A: new GPU tests, BRC full capture (source-level), C4 batch FP64 op counts.
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests/test_reference_shim.py tests/test_gpu_big.py -m gpu -q -rf > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/pytest_new.log
bash tools/ncu_brc.sh r2a_brc_full 10000000
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
for w in brc_batch worst_off_batch; do
  CMD="python bench.py --workload $w --steps 1 --warmup 1 --paths-per-gpu 200000 --e2e-steps 0 --no-cpu-baseline"
  $CMD > $O/plain_$w.log 2>&1 && ncu --metrics $M --clock-control none -k regex:path -s 1 -c 1 --csv --log-file $O/fp64ops_$w.csv $CMD > $O/ncu_$w.log 2>&1
  echo "$w rc=$?" >> $O/fp64ops.rc
done
echo done
