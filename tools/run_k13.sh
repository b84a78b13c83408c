mkdir -p gpurun_out
timeout 120 python tools/probe_k13.py > gpurun_out/k13p.log 2>&1 || { echo "probe failed/hung $?" >> gpurun_out/k13p.log; exit 1; }
timeout 60 python tools/bench_k13.py > gpurun_out/k13.log 2>&1
timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_tucker.py tests/test_gpu_tucker_factors.py -m gpu -q -x > gpurun_out/t_k13.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_k13.log
