#!/bin/bash
# NVRTC-kernel variants by extra NVRTC flags (run under gpurun):
#   tools/jitvar.sh "" "-DCLTK_PHASE_UNROLL=2" ...
for fl in "$@"; do
  r=$(CLTK_JIT_FLAGS="$fl" timeout 300 python bench.py --steps 3 --warmup 2 --paths-per-gpu 20000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))")
  echo "[$fl] $r"
done
