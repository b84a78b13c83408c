python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-extra > gpurun_out/res.json 2>gpurun_out/res.err
KS_GRAPH_TIMELINE=1 python tools/graph_timeline.py > gpurun_out/tl.log 2>&1
KS_GRAPH_TIMELINE=1 python tools/graph_timeline.py --host > gpurun_out/tlh.log 2>&1
