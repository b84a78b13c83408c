mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_dense.py tests/test_gpu_tucker.py tests/test_gpu_tucker_factors.py tests/test_gpu_solvers.py tests/test_gpu_baselines.py -m gpu -q -x > gpurun_out/t_core.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_core.log
timeout 200 python tools/profile_core.py > gpurun_out/core.log 2>&1
