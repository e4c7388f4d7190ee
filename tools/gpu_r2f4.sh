#!/bin/bash
# host-side trace of the e2e calls of the short workloads
O=gpurun_out; mkdir -p $O
for w in "worst_off 16000000" "call 100000000" "worst_off_batch 2000000"; do
  set -- $w
  CLTK_TRACE=1 python bench.py --workload $1 --paths-per-gpu $2 --steps 2 --warmup 3 --e2e-steps 4 --no-cpu-baseline > $O/e2e_$1.json 2> $O/e2e_$1.err
  echo "== $1"; grep cltk $O/e2e_$1.err | tail -6
  python -c "import json; d=json.loads(open('$O/e2e_$1.json').read().strip().splitlines()[-1]); print(d['e2e']['samples_ms'], d['config']['kernel_ms'], d['ms_per_step'])"
done
