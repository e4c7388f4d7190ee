# batch-size variants (CLTK_MAX_BATCH 6 / 9 / 12) on the BRC and worst-off
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_y.txt
run() { r=$(CLTK_B200_LIB=$2 CLTK_JIT_CACHE_DIR=/tmp/jc_$1 timeout 300 python bench.py --workload $3 --steps 3 --warmup 2 --paths-per-gpu $4 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $3 $r" >> $O/var_y.txt; }
for i in 1 2; do
for v in 6 9 12; do
  lib=$PWD/build/variants/b$v/libcltk_b200.so; [ $v = 6 ] && lib=$PWD/paper_2108_03076_b200/libcltk_b200.so
  run b$v $lib brc 20000000
done
done
for v in 6 9 12; do
  lib=$PWD/build/variants/b$v/libcltk_b200.so; [ $v = 6 ] && lib=$PWD/paper_2108_03076_b200/libcltk_b200.so
  run b$v $lib worst_off 16000000
done
echo done
