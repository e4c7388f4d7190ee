#!/bin/bash
# call / fx / BRC: current engine vs the previous build (libcltk_b200_old.so), under gpurun
run() { timeout 300 python bench.py --workload $1 --steps 5 --warmup 3 --paths-per-gpu $2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%s %.4g %r' % ('$1', d['value'], d['price']))"; }
for i in 1 2; do
  echo "new:"; run call 100000000; run brc 20000000
  mv paper_2108_03076_b200/libcltk_b200.so /tmp/new.so; cp paper_2108_03076_b200/libcltk_b200_old.so paper_2108_03076_b200/libcltk_b200.so
  echo "old:"; run call 100000000; run brc 20000000
  mv /tmp/new.so paper_2108_03076_b200/libcltk_b200.so
done
