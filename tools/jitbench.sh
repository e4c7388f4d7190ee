#!/bin/bash
# interpreter vs NVRTC payoff kernel on the bench workloads (run under gpurun)
for w in brc brc_batch worst_off; do
  case $w in brc) P=50000000;; brc_batch) P=5000000;; worst_off) P=16000000;; esac
  for j in 0 1; do
    r=$(timeout 600 python bench.py --workload $w --jit $j --steps 3 --warmup 3 --paths-per-gpu $P --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g e2e %.4g price %r jit %s' % (d['value'], d['e2e']['value'], d['price'], d['plan']['jit']))")
    echo "$w jit=$j $r"
  done
done
