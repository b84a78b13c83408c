mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_dense.py tests/test_gpu_c4.py tests/test_gpu_tucker.py -m gpu -q -x > gpurun_out/t_k2.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_k2.log
timeout 200 python tools/probe_k2.py > gpurun_out/k2_new.log 2>&1
(cd _ab/base && timeout 200 python tools/probe_k2.py > ../../gpurun_out/k2_base.log 2>&1)
