set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
: > $O/var_k.txt
run() { r=$(timeout 300 python bench.py --workload $2 --steps 3 --warmup 2 --paths-per-gpu $3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))"); echo "$1 $2 $r" >> $O/var_k.txt; }
run new worst_off_batch 2000000
CLTK_B200_LIB=$PWD/build/variants/old/libcltk_b200.so run old worst_off_batch 2000000
run new brc_batch 2000000
CLTK_B200_LIB=$PWD/build/variants/old/libcltk_b200.so run old brc_batch 2000000
