#!/bin/bash
# streamed copy-out (row stages): layout tests, stage-schedule sweep, trace
cd /root/repo
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/gpu_layout.txt 2>&1; echo "exit $?" >> gpurun_out/gpu_layout.txt
for sc in "" "1024,1536,2048,2560,3072,3584,3072,2048,1024" "1024,1536,2048,2560,3072,4096,5664" "1024,2048,3072,3584,3584,3584,2048,1024" "1536,2560,3584,4096,4096,3072,1024" "1024,1536,2048,2560,3072,3584,2560,1536,1024,512"; do
  PS_STAGE_COLS="$sc" timeout 300 python tools/e2e_probe.py c5 2>/dev/null | tail -1 >> gpurun_out/e2e_sweep4.jsonl
done
PS_PIPE_TRACE=2 timeout 300 python tools/e2e_probe.py c5 > gpurun_out/e2e_trace_rows.txt 2>&1
