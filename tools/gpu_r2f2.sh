#!/bin/bash
# A/B: long-path step loop batch-major (CLTK_SIM_LOOP 1 / 2) vs step-major
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_f2.txt
for i in 1 2; do
bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_SIM_LOOP=1" "-DCLTK_SIM_LOOP=2" >> $O/var_f2.txt 2>&1
done
echo done
