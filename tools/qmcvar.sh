#!/bin/bash
# QMC NVRTC-kernel variants by extra NVRTC flags (run under gpurun)
for fl in "$@"; do
  r=$(CLTK_JIT_FLAGS="$fl" timeout 300 python bench.py --rng sobol --steps 3 --warmup 2 --paths-per-gpu 20000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %r' % (d['value'], d['price']))")
  echo "[$fl] $r"
done
