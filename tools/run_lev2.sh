mkdir -p gpurun_out
timeout 200 python tools/probe_lev.py > gpurun_out/lev.log 2>&1
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_solvers.py tests/test_gpu_sampling.py tests/test_gpu_dense.py tests/test_gpu_tucker.py -m gpu -q -x > gpurun_out/t_lev.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_lev.log
KS_GRAPH_TIMELINE=1 timeout 400 python tools/graph_timeline.py --c4 > gpurun_out/tl_c4.log 2>&1
