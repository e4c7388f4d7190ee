#!/bin/bash
# Round-2 final build: full ncu captures of the three Philox workloads' path
# kernels and the launch list of the default bench command (run under gpurun).
set -u
O=gpurun_out
mkdir -p $O
bash tools/ncu_brc.sh brc_full 10000000
bash tools/ncu_wl.sh wo_full worst_off 4000000
bash tools/ncu_wl.sh call_full call 40000000
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "launches rc=$?"
