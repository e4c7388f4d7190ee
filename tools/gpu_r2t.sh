set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_jit.py -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
: > $O/var_t.txt
run() { r=$(CLTK_JIT_CACHE_DIR=/tmp/jc_$1 timeout 300 python bench.py --workload $2 --steps 3 --warmup 2 --paths-per-gpu $3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $2 $r" >> $O/var_t.txt; }
for i in 1 2; do
run new brc 20000000
CLTK_B200_LIB=$PWD/build/variants/old/libcltk_b200.so run old brc 20000000
done
