mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -k "exact" > gpurun_out/t_exact.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_exact.log
timeout 400 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_tucker_factors.py tests/test_gpu_tucker_props.py tests/test_gpu_baselines.py tests/test_gpu_dense.py tests/test_gpu_c4.py -m gpu -q -x >> gpurun_out/t_exact.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_exact.log
timeout 200 python tools/profile_core.py > gpurun_out/core.log 2>&1
