#!/bin/bash
# NVRTC-kernel variants for one workload (run under gpurun): tools/wlvar.sh WORKLOAD PATHS "flags"...
w=$1; n=$2; shift 2
for fl in "$@"; do
  r=$(CLTK_JIT_FLAGS="$fl" timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --paths-per-gpu $n --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %r' % (d['value'], d['price']))")
  echo "[$w $fl] $r"
done
