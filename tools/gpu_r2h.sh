set -u
O=gpurun_out; mkdir -p $O
: > $O/var_h.txt
run() { r=$(timeout 300 python bench.py --workload brc --steps 3 --warmup 2 --paths-per-gpu 20000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])"); echo "$1 $r" >> $O/var_h.txt; }
for i in 1 2; do
  run new
  CLTK_B200_LIB=$PWD/build/variants/old/libcltk_b200.so run old
  CLTK_B200_LIB=$PWD/build/variants/old/libcltk_b200.so CLTK_JIT_FLAGS="-DCLTK_P1_UNROLL=6" run old_u6
done
