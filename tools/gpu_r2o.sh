set -u
O=gpurun_out; mkdir -p $O
: > $O/var_o.txt
run() { r=$(CLTK_JIT_CACHE_DIR=/tmp/jc_$1 timeout 300 python bench.py --workload $2 --steps 3 --warmup 2 --paths-per-gpu $3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $2 $r" >> $O/var_o.txt; }
for v in b64 b256; do
  if [ -f build/variants/$v/libcltk_b200.so ]; then
    CLTK_JIT_CACHE_DIR=/tmp/jc_t$v CLTK_B200_LIB=$PWD/build/variants/$v/libcltk_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_jit.py -m gpu -q -x > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
  fi
done
for i in 1 2; do
  run b128 brc 20000000
  for v in b64 b256; do [ -f build/variants/$v/libcltk_b200.so ] && CLTK_B200_LIB=$PWD/build/variants/$v/libcltk_b200.so run $v brc 20000000; done
done
run b128 worst_off 16000000
for v in b64 b256; do [ -f build/variants/$v/libcltk_b200.so ] && CLTK_B200_LIB=$PWD/build/variants/$v/libcltk_b200.so run $v worst_off 16000000; done
run b128 call 100000000
for v in b64 b256; do [ -f build/variants/$v/libcltk_b200.so ] && CLTK_B200_LIB=$PWD/build/variants/$v/libcltk_b200.so run $v call 100000000; done
