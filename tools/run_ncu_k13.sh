mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kron3_ -c 1 -o gpurun_out/k13 python tools/bench_k13.py > gpurun_out/ncu_k13.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_k13.log
