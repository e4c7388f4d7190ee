#!/bin/bash
# CLI price twice in fresh processes with an empty on-disk NVRTC cache: the
# second run loads the cubin instead of compiling (run under gpurun).
export CLTK_JIT_CACHE_DIR=/tmp/cltk_cache_test; rm -rf $CLTK_JIT_CACHE_DIR
for i in 1 2; do
  s=$(date +%s.%N)
  python -m paper_2108_03076_b200 price tests/golden/kernels/brc.json --model tests/golden/models/three.json \
    --paths 1000000 --seed 42 > gpurun_out/cli$i.json
  e=$(date +%s.%N)
  python3 -c "print('cli run $i: %.2f s' % ($e - $s))"
done
ls -la $CLTK_JIT_CACHE_DIR
