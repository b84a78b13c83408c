# Round-end evidence: the full GPU suite, the default bench line, the reference arm, the ncu launch list
# of the bench command, ncu --set full of the persistent loop kernel and of the K13 kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --skip-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:richardson_phased_kernel -c 1 -o gpurun_out/loop python tools/profile_fast.py c3 3 > gpurun_out/ncu_loop.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kron3_ -c 1 -o gpurun_out/k13 python tools/bench_k13.py > gpurun_out/ncu_k13.log 2>&1
