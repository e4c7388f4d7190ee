#!/bin/bash
# A/B: register budget of the NVRTC kernel (resident CTAs per SM: 8 = 64 registers)
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_f3.txt
for i in 1 2; do
bash tools/jitvar_wl.sh call 100000000 "" "-DCLTK_MIN_BLOCKS=7" "-DCLTK_MIN_BLOCKS=6" >> $O/var_f3.txt 2>&1
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_MIN_BLOCKS=7" "-DCLTK_MIN_BLOCKS=6" >> $O/var_f3.txt 2>&1
bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_MIN_BLOCKS=7" >> $O/var_f3.txt 2>&1
done
echo done
