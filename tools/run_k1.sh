mkdir -p gpurun_out
for i in 1 2; do
timeout 200 python tools/probe_k2.py n=16384 64 > gpurun_out/k1_new_$i.log 2>&1
(cd _ab/base && timeout 200 python tools/probe_k2.py n=16384 64 > ../../gpurun_out/k1_base_$i.log 2>&1)
done
