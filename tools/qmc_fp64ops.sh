#!/bin/bash
# FP64 SASS op counts of the QMC (Sobol) BRC kernel -> its own F_path (run under gpurun)
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
CMD="python bench.py --rng sobol --steps 1 --warmup 1 --paths-per-gpu 2000000 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_qmc.log 2>&1 && ncu --metrics $M --clock-control none -k regex:path -s 1 -c 1 --csv --log-file gpurun_out/fp64ops_qmc.csv $CMD > gpurun_out/ncu_qmc.log 2>&1
echo "rc=$?"
