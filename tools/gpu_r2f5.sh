#!/bin/bash
# A/B: stream loop as nested 32-bit loops + per-chunk active count (new) vs HEAD (base)
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_f5.txt
B=build/variants/base/libcltk_b200.so; N=paper_2108_03076_b200/libcltk_b200.so
bash tools/ablib.sh $B $N call 100000000 2 >> $O/var_f5.txt 2>&1
bash tools/ablib.sh $B $N worst_off 16000000 2 >> $O/var_f5.txt 2>&1
bash tools/ablib.sh $B $N brc 20000000 1 >> $O/var_f5.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -rf > $O/pytest_f5.log 2>&1; echo "pytest rc=$?" >> $O/pytest_f5.log
echo done
