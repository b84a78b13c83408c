mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_c4.py -m gpu -q -x > gpurun_out/t_fetch.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_fetch.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --skip-cpu > gpurun_out/b_new$i.json 2>/dev/null
KS_FETCH_OUTSIDE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --skip-cpu > gpurun_out/b_old$i.json 2>/dev/null
done
