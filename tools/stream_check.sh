#!/bin/bash
# row-stage schedule variants (first stage width), then the bench line and the reference arm
cd /root/repo
mkdir -p gpurun_out
for sc in "" "512,1024,2048,3072,3584,3584,3584,2080,1024" "512,1536,2560,3584,3584,3584,2560,1536,512" "1024,2048,3072,4096,4096,3072,2048,512"; do
  PS_STAGE_COLS="$sc" timeout 300 python tools/e2e_probe.py c5 2>/dev/null | tail -1 >> gpurun_out/e2e_sweep6.jsonl
done
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err
