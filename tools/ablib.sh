#!/bin/bash
# A/B of two engine libraries (run under gpurun):
#   tools/ablib.sh <libA> <libB> <workload> <paths> [rounds]
a=$1; b=$2; wl=$3; n=$4; rounds=${5:-2}
for i in $(seq $rounds); do
  for lib in $a $b; do
    r=$(CLTK_B200_LIB=$lib timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --paths-per-gpu $n --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'] or 0, d['price']))")
    echo "$wl [$lib] $r"
  done
done
