set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_jit.py tests/test_gpu_faults.py tests/test_gpu_big.py -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
: > $O/var_i.txt
run() { r=$(timeout 300 python bench.py --workload brc --steps 3 --warmup 2 --paths-per-gpu 20000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %r' % (d['value'], d['price']))"); echo "$1 $r" >> $O/var_i.txt; }
for i in 1 2; do
  run prefetch
  CLTK_JIT_FLAGS="-DCLTK_PREFETCH=0" run noprefetch
  CLTK_JIT_FLAGS="-DCLTK_P5_UNROLL=3" run prefetch_u3
  CLTK_JIT_FLAGS="-DCLTK_P5_UNROLL=6" run prefetch_u6
done
