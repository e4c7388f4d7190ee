set -u
O=gpurun_out; mkdir -p $O
bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_ONE_BARRIER_PAIR=1" "-DCLTK_ONE_BARRIER_PAIR=1 -DCLTK_R2_ROT=0" "-DCLTK_ONE_BARRIER_PAIR=1 -DCLTK_R2_ROT=1" "-DCLTK_ONE_BARRIER_PAIR=1 -DCLTK_R2_ROT=3" "-DCLTK_P1_UNROLL=1" "-DCLTK_P3_UNROLL=3" "-DCLTK_P5_UNROLL=3" "-DCLTK_P3_UNROLL=1" > $O/var_brc2.txt 2>&1
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_ONE_BARRIER_PAIR=1" > $O/var_wo2.txt 2>&1
