#!/bin/bash
# Full ncu capture of the C4 batch path kernel (run under gpurun): gpurun_out/$1.ncu-rep
name=${1:-batch_full}
CMD="python bench.py --workload brc_batch --steps 1 --warmup 3 --paths-per-gpu 1000000 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${name}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path -s 3 -c 1 \
  -o gpurun_out/$name $CMD > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"
