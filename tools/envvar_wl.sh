#!/bin/bash
# Variants by environment assignments for one workload (run under gpurun):
#   tools/envvar_wl.sh <workload> <paths> "" "CLTK_JIT_MAX_CARRY=0" "CLTK_JIT_FLAGS=-DX=1" ...
wl=$1; n=$2; shift 2
for ev in "$@"; do
  r=$(env $ev timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --paths-per-gpu $n --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'] or 0, d['price']))")
  echo "$wl [$ev] $r"
done
