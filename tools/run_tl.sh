mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_solvers.py tests/test_gpu_c4.py -m gpu -q -x > gpurun_out/t_tl.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_tl.log
KS_GRAPH_TIMELINE=1 timeout 200 python tools/graph_timeline.py > gpurun_out/tl.log 2>&1
KS_GRAPH_TIMELINE=1 timeout 400 python tools/graph_timeline.py --c4 > gpurun_out/tl_c4.log 2>&1
