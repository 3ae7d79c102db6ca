#!/bin/bash
# Per-config bench lines (device value + e2e) for BASELINE.md 6 / profiles:
# C1-C5 split, plus FP64-mode lines for C3 and C5.  Run on the GPU box.
out=${1:-gpurun_out/r02_configs}
mkdir -p "$out"
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
for c in c3 c5; do
  python bench.py --config $c --precision fp64 --steps 3 --warmup 3 --no-cpu > "$out/bench_${c}_fp64.json" 2> "$out/bench_${c}_fp64.err"
done
