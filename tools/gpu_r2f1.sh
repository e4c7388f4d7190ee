#!/bin/bash
# A/B: Acklam tails dealt within the warp (two barriers per batch instead of four)
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_f1.txt
for i in 1 2; do
bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_TAIL_POOL=0" "-DCLTK_CTA_POOL=0" >> $O/var_f1.txt 2>&1
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_TAIL_POOL=0" >> $O/var_f1.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" "-DCLTK_TAIL_POOL=0" >> $O/var_f1.txt 2>&1
done
echo done
