#!/bin/bash
# NVRTC-kernel variants by extra NVRTC flags for one workload (run under gpurun):
#   tools/jitvar_wl.sh <workload> <paths> "" "-DX=1" ...
wl=$1; n=$2; shift 2
for fl in "$@"; do
  r=$(CLTK_JIT_FLAGS="$fl" timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --paths-per-gpu $n --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'] or 0, d['price']))")
  echo "$wl [$fl] $r"
done
