mkdir -p gpurun_out
timeout 200 python tools/probe_lev.py > gpurun_out/lev.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lev_launches.csv python tools/probe_lev.py 65536 64 3 > gpurun_out/lev_ncu.log 2>&1
