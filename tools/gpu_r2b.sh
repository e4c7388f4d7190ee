set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
bash tools/jitvar_wl.sh brc 20000000 "" "-DCLTK_MERGED_PASS=0" "-DCLTK_R2_ROT=1" "-DCLTK_R2_ROT=2" "-DCLTK_R2_ROT=3" "-DCLTK_R3_ROT=1" "-DCLTK_R3_ROT=3" > $O/var_brc.txt 2>&1
bash tools/jitvar_wl.sh worst_off 16000000 "" "-DCLTK_MERGED_PASS=0" > $O/var_wo.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" "-DCLTK_MERGED_PASS=0" > $O/var_call.txt 2>&1
