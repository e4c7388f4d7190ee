set -u
O=gpurun_out; mkdir -p $O
: > $O/var_u.txt
run() { r=$(CLTK_JIT_CACHE_DIR=/tmp/jc_$1 timeout 300 python bench.py --workload $2 --steps 3 --warmup 2 --paths-per-gpu $3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $2 $r" >> $O/var_u.txt; }
for i in 1 2; do
run base brc 20000000
CLTK_JIT_FLAGS="-DCLTK_MIN_BLOCKS=7" run mb7 brc 20000000
CLTK_JIT_FLAGS="-DCLTK_MIN_BLOCKS=6" run mb6 brc 20000000
done
run base worst_off 16000000
CLTK_JIT_FLAGS="-DCLTK_MIN_BLOCKS=7" run mb7 worst_off 16000000
