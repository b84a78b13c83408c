mkdir -p gpurun_out
timeout 200 python bench.py --steps 20 --warmup 5 --no-extra --skip-cpu ${AB_ARGS} > gpurun_out/ab_new_1.json 2> gpurun_out/ab_new_1.err
