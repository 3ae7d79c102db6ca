#!/bin/bash
# Round-2 closing measurements on the GPU box: per-config bench lines (device
# value + e2e) for C1-C5 split and C3/C5 FP64, the Gauss-forced C2/C4 check,
# the time-resolved probe, then the C5 launch list and one full ncu capture of
# its Gram (each after its own command ran clean without ncu).
out=${1:-gpurun_out/r02_final}
mkdir -p "$out"
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
for c in c3 c5; do
  python bench.py --config $c --precision fp64 --steps 3 --warmup 3 --no-cpu > "$out/bench_${c}_fp64.json" 2> "$out/bench_${c}_fp64.err"
done
for c in c2 c4; do
  PS_GAUSS=1 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > "$out/bench_${c}_gauss.json" 2>/dev/null
done
for a in "2048 256 128 full" "2048 256 128 upper" "4096 64 256 full"; do
  python tools/over_trials_probe.py $a >> "$out/over_trials.txt" 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > "$out/plain.log" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/c5_launches.csv" $CMD > "$out/ncu_launch.log" 2>&1
$CMD > "$out/plain2.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gram_split -s 3 -c 1 -o "$out/c5_gram" $CMD > "$out/ncu_full.log" 2>&1
echo done >> "$out/done.txt"
