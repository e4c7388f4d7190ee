# stream kernels (worst-off, call): phase-unroll variants (NVRTC flags)
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_ac.txt
for i in 1 2; do
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_P1_UNROLL=3" "-DCLTK_P1_UNROLL=6" "-DCLTK_P5_UNROLL=6" "-DCLTK_P5_UNROLL=3" "-DCLTK_P1_UNROLL=1" >> $O/var_ac.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" "-DCLTK_P1_UNROLL=3" "-DCLTK_P1_UNROLL=6" "-DCLTK_P5_UNROLL=6" "-DCLTK_P5_UNROLL=3" "-DCLTK_P1_UNROLL=1" >> $O/var_ac.txt 2>&1
done
echo done
