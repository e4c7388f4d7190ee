#!/bin/bash
# One GPU session: parity suite, benches of every config, FP64 op counts.
# Writes gpurun_out/*.log|json.  Usage (under gpurun): bash tools/gpu_round.sh [quick]
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_brc.json 2> $O/bench_brc.err
timeout 600 python bench.py --workload worst_off --paths-per-gpu 16000000 --ref-paths 200000 > $O/bench_worst_off.json 2> $O/bench_worst_off.err
timeout 600 python bench.py --workload call --paths-per-gpu 100000000 --ref-paths 4000000 > $O/bench_call.json 2> $O/bench_call.err
timeout 900 python bench.py --workload brc_batch --paths-per-gpu 10000000 --e2e-steps 1 > $O/bench_brc_batch.json 2> $O/bench_brc_batch.err
timeout 900 python bench.py --workload worst_off_batch --paths-per-gpu 2000000 --e2e-steps 1 > $O/bench_worst_off_batch.json 2> $O/bench_worst_off_batch.err
timeout 600 python bench.py --rng sobol --paths-per-gpu 50000000 --no-cpu-baseline > $O/bench_brc_qmc.json 2> $O/bench_brc_qmc.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 1 > $O/bench_gpus2.json 2> $O/bench_gpus2.err; echo "rc=$?" >> $O/bench_gpus2.err
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
for w in worst_off call; do
  CMD="python bench.py --workload $w --steps 1 --warmup 1 --paths-per-gpu 2000000 --e2e-steps 0 --no-cpu-baseline"
  $CMD > $O/plain_$w.log 2>&1 && ncu --metrics $M --clock-control none -k regex:path -s 1 -c 1 --csv --log-file $O/fp64ops_$w.csv $CMD > $O/ncu_$w.log 2>&1
done
if [ "${1:-}" = "full" ]; then
  # launch list of the default bench command (per-launch times, cold-cache, serialised)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
  # one full capture of the hot kernel (smaller step so the ~40 replays stay short)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path -s 3 -c 1 \
    -o $O/brc_full python bench.py --steps 1 --warmup 3 --paths-per-gpu 10000000 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
  bash tools/ncu_wl.sh wo_full worst_off 4000000
  bash tools/ncu_wl.sh call_full call 40000000
  bash tools/ncu_qmc.sh qmc_full
fi
echo done
