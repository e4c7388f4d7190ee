#!/bin/bash
# A/B: log-domain spots on/off (env), 20M paths
for v in on off on off; do
  if [ $v = off ]; then export CLTK_JIT_NO_LOGSPOTS=1; else unset CLTK_JIT_NO_LOGSPOTS; fi
  r=$(timeout 300 python bench.py --steps 3 --warmup 2 --paths-per-gpu 20000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))")
  echo "[logspots $v] $r"
done
