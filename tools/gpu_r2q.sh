set -u
O=gpurun_out; mkdir -p $O
: > $O/var_q.txt
run() { r=$(CLTK_JIT_CACHE_DIR=/tmp/jc_$1 timeout 300 python bench.py --workload $2 --steps 3 --warmup 2 --paths-per-gpu $3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $2 $r" >> $O/var_q.txt; }
for i in 1 2; do
run new brc 20000000
CLTK_B200_LIB=$PWD/build/variants/ma4/libcltk_b200.so run ma4 brc 20000000
done
run new worst_off 16000000
CLTK_B200_LIB=$PWD/build/variants/ma4/libcltk_b200.so run ma4 worst_off 16000000
