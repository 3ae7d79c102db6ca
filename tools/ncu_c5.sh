#!/bin/bash
# launch list + one full capture of the Gram for the bench workload (C5), and the GPU parity log
cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rA > gpurun_out/gpu_parity.txt 2>&1; echo "tests exit $?" >> gpurun_out/gpu_parity.txt
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_split -s 3 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
