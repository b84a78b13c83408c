mkdir -p gpurun_out
timeout 120 python tools/probe_tables.py > gpurun_out/tables.log 2>&1
KS_TABLES_ONE_CTA=1 timeout 120 python tools/probe_tables.py > gpurun_out/tables_1cta.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_api_units.py tests/test_gpu_c4.py tests/test_gpu_solvers.py -m gpu -q -x > gpurun_out/t_tab.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_tab.log
KS_GRAPH_TIMELINE=1 timeout 400 python tools/graph_timeline.py --c4 > gpurun_out/tl_c4.log 2>&1
