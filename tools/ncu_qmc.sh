#!/bin/bash
# Full ncu capture of the QMC (Sobol) BRC path kernel (run under gpurun): gpurun_out/$1.ncu-rep
name=${1:-qmc_full}
CMD="python bench.py --rng sobol --steps 1 --warmup 3 --paths-per-gpu 10000000 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${name}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path -s 3 -c 1 \
  -o gpurun_out/$name $CMD > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"
