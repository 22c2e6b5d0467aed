#!/bin/bash
# End-of-round refresh: tests, smoke, every bench line, C5 at full size, stream
# and simulate modes, reference arm, launch list, torchrun N = 1.
bash tools/refresh_r02b.sh
out=gpurun_out/refresh
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_c5_full.jsonl 2>&1
rm -f $out/stream.jsonl $out/simulate.jsonl
for c in C1 T1-R1/4 T1-R1/2 T1-R3/4 C2 C3-R1/2 C4 C5; do timeout 200 python bench.py --mode stream --config $c >> $out/stream.jsonl 2>&1; done
for c in C4 C2 C1; do timeout 300 python bench.py --mode simulate --config $c --steps 3 --warmup 3 >> $out/simulate.jsonl 2>&1; done
tail -2 $out/smoke.log; grep -h '^{' $out/bench_c5_full.jsonl | cut -c1-200
