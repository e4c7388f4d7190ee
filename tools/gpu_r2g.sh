set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
bash tools/envvar_wl.sh brc 20000000 "A=1" "A=2" > $O/var_g.txt 2>&1
bash tools/envvar_wl.sh worst_off 16000000 "A=1" >> $O/var_g.txt 2>&1
