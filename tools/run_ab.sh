# A/B against the committed state (_ab/base, built from git HEAD): hang-guarded checks, the solve-path
# tests, then alternating bench runs of both trees
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t_ab.log 2>&1 || { echo "smoke failed/hung $?" >> gpurun_out/t_ab.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -k "c3" >> gpurun_out/t_ab.log 2>&1 || { echo "c3 failed/hung $?" >> gpurun_out/t_ab.log; exit 1; }
timeout 600 python -m pytest ${AB_TESTS:-tests/test_gpu_solvers.py tests/test_gpu_c4.py tests/test_gpu_distributed.py} -m gpu -q -x >> gpurun_out/t_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_ab.log
for i in 1 2; do
timeout 200 python bench.py --steps 20 --warmup 5 --no-extra --skip-cpu ${AB_ARGS} > gpurun_out/ab_new_$i.json 2> gpurun_out/ab_new_$i.err
(cd _ab/base && timeout 200 python bench.py --steps 20 --warmup 5 --no-extra --skip-cpu ${AB_ARGS} > ../../gpurun_out/ab_base_$i.json 2> ../../gpurun_out/ab_base_$i.err)
done
