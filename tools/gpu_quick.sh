#!/bin/bash
# Quick GPU session: the GPU test suite (or a subset), the smoke, one default
# bench line.  Usage (under gpurun): bash tools/gpu_quick.sh [pytest -k expr]
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
K=${1:-}
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "$K" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
else
  timeout 1800 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_brc.json 2> $O/bench_brc.err; echo "bench rc=$?" >> $O/bench_brc.err
timeout 120 python bench.py --gpus 2 --steps 1 --warmup 1 > $O/bench_gpus2.json 2> $O/bench_gpus2.err; echo "bench2 rc=$?" >> $O/bench_gpus2.err
echo done
