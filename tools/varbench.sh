for d in build/variants/*/; do
  r=$(CLTK_B200_LIB=$PWD/${d}libcltk_b200.so timeout 300 python bench.py --steps 3 --warmup 1 --paths-per-gpu 10000000 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f %r' % (d['value'], d['roofline']['frac'], d['price']))")
  echo "$d $r"
done
