# NVRTC-only variants of the BRC kernel: phase unrolls
set -u
O=gpurun_out; mkdir -p $O
: > $O/var_z.txt
for i in 1 2; do
  bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=6" "-DCLTK_P3_UNROLL=6" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=3" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=6 -DCLTK_P1_UNROLL=6" >> $O/var_z.txt 2>&1
done
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=6" "-DCLTK_P3_UNROLL=6" >> $O/var_z.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=6" "-DCLTK_P3_UNROLL=6" >> $O/var_z.txt 2>&1
bash tools/jitvar_wl.sh brc_batch 4000000 "" "-DCLTK_P3_UNROLL=6 -DCLTK_P5_UNROLL=6" >> $O/var_z.txt 2>&1
echo done
