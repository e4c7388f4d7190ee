# stream phase-1 unroll 3 for multi-asset streams: parity + benches
set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_ad.log 2>&1; echo "pytest rc=$?" >> $O/pytest_ad.log
: > $O/var_ad.txt
for i in 1 2; do
bash tools/jitvar_wl.sh worst_off 16000000 "" >> $O/var_ad.txt 2>&1
bash tools/jitvar_wl.sh worst_off_batch 2000000 "" >> $O/var_ad.txt 2>&1
bash tools/jitvar_wl.sh call 100000000 "" >> $O/var_ad.txt 2>&1
done
echo done
