# long-path unrolls adopted: parity + the bench lines
set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_aa.log 2>&1; echo "pytest rc=$?" >> $O/pytest_aa.log
: > $O/var_aa.txt
for i in 1 2; do bash tools/jitvar_wl.sh brc 20000000 "" >> $O/var_aa.txt 2>&1; done
bash tools/jitvar_wl.sh worst_off 16000000 "" >> $O/var_aa.txt 2>&1
bash tools/jitvar_wl.sh brc_batch 4000000 "" >> $O/var_aa.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" >> $O/var_aa.txt 2>&1
echo done
