#!/bin/bash
# exit-as-value log-domain extrema (new) vs HEAD (base): template batches; GPU suite
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_f6.txt
B=build/variants/base/libcltk_b200.so; N=paper_2108_03076_b200/libcltk_b200.so
bash tools/ablib.sh $B $N brc_batch 5000000 2 >> $O/var_f6.txt 2>&1
bash tools/ablib.sh $B $N worst_off_batch 2000000 1 >> $O/var_f6.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_f6.log 2>&1; echo "pytest rc=$?" >> $O/pytest_f6.log
echo done
