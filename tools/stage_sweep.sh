#!/bin/bash
# e2e stage-schedule sweep on C5 (upper layout): one JSON line per schedule
cd /root/repo
PS_PIPE_TRACE=1 python tools/e2e_probe.py c5 > gpurun_out/e2e_trace_default.txt 2>&1
PS_PIPE_TRACE=1 PS_PIPE_NO_D2H=1 python tools/e2e_probe.py c5 > gpurun_out/e2e_trace_nod2h.txt 2>&1
for sc in "1024" "2048" "1024,1536,2048,2560,3072,3072,2560,2048,1536,1024" "1024,1536,2048,2560,2560,2560,2048,1536,1024,512" "512,1024,1536,2048,2048,2048,2048,2048,1536,1024,512,512" "1024,2048,3072,3072,3072,2048,1024,1024,1024,1024,1024"; do
  PS_STAGE_COLS="$sc" python tools/e2e_probe.py c5 2>/dev/null | tail -1 >> gpurun_out/e2e_sweep.jsonl
done
PS_PIPE_TRACE=1 PS_STAGE_COLS="1024,1536,2048,2560,2560,2560,2048,1536,1024,512" python tools/e2e_probe.py c5 > gpurun_out/e2e_trace_shrink.txt 2>&1
