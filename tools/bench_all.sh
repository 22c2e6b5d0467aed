#!/bin/bash
# Run bench.py over every BASELINE.json config (reduced frame counts where the
# full config would take minutes) and append the JSON lines to $1.
out=${1:-gpurun_out/cfg.log}
shift
rm -f "$out"
for c in C1:1000 C2:10000 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:200000 C5:16384 T1-R1/4:1000 T1-R1/2:1000 T1-R3/4:1000 T1-R1/4:100000 T1-R1/2:100000 T1-R3/4:100000; do
  cfg=${c%%:*}; fr=${c##*:}
  timeout 300 python bench.py --config $cfg --frames $fr --steps 3 --warmup 3 --no-cpu-baseline "$@" >> "$out" 2>&1
done
