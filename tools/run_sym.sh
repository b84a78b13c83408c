mkdir -p gpurun_out
timeout 200 python tools/probe_lev.py > gpurun_out/lev.log 2>&1
timeout 1100 python -m pytest tests -m gpu -q -x > gpurun_out/t_sym.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_sym.log
KS_GRAPH_TIMELINE=1 timeout 400 python tools/graph_timeline.py --c4 > gpurun_out/tl_c4.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --skip-cpu > gpurun_out/b_new$i.json 2>/dev/null
KS_TALL_OLD=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --skip-cpu > gpurun_out/b_old$i.json 2>/dev/null
done
