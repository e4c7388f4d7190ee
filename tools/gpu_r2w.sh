# instance-major pairs: batch/JIT parity tests, then the C4 bench lines
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_jit.py tests/test_gpu_parity.py -m gpu -q -rf -x > $O/pytest_w.log 2>&1; echo "pytest rc=$?" >> $O/pytest_w.log
for i in 1 2; do
timeout 300 python bench.py --workload worst_off_batch --paths-per-gpu 2000000 --no-cpu-baseline > $O/w_wob_$i.json 2> $O/w_wob_$i.err
timeout 300 python bench.py --workload brc_batch --paths-per-gpu 10000000 --no-cpu-baseline > $O/w_brcb_$i.json 2> $O/w_brcb_$i.err
done
echo done
