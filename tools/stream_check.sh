#!/bin/bash
# streamed copy-out (row stages): band sizes (all stages / final stage)
cd /root/repo
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/gpu_layout.txt 2>&1; echo "exit $?" >> gpurun_out/gpu_layout.txt
for bl in "4 4" "4 2" "4 1" "2 1" "6 2" "8 2"; do
  set -- $bl
  PS_SB_BAND=$1 PS_SB_BAND_LAST=$2 timeout 300 python tools/e2e_probe.py c5 2>/dev/null | tail -1 >> gpurun_out/e2e_sweep5.jsonl
done
