#!/bin/bash
# Full ncu capture of one workload's path kernel (run under gpurun):
#   tools/ncu_wl.sh <name> <workload> <paths>  -> gpurun_out/<name>.ncu-rep
name=$1; wl=$2; paths=$3
CMD="python bench.py --workload $wl --steps 1 --warmup 3 --paths-per-gpu $paths --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${name}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path -s 3 -c 1 \
  -o gpurun_out/$name $CMD > gpurun_out/${name}_ncu.log 2>&1
echo "$name ncu rc=$?"
