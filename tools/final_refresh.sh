#!/bin/bash
# One GPU call refreshing every committed measurement of round 2:
# issue profile, one bench line per workload, the default bench line, the
# reference arm, stream / simulate modes, an ncu launch list of the default
# bench and ncu --set full captures of the C4 and C5 bench launches.
out=gpurun_out/final; mkdir -p $out
timeout 2400 python tools/issue_profile.py $out/issue.json > $out/issue.log 2>&1 && cp $out/issue.json profiles/issue.json
bash tools/bench_all.sh $out/all_configs.jsonl
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_c5_full.jsonl 2>&1
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_c2_sweep.jsonl 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_default.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.jsonl 2>&1
for c in C1 T1-R1/4 T1-R1/2 T1-R3/4 C2 C3-R1/2 C4 C5; do timeout 200 python bench.py --mode stream --config $c >> $out/stream.jsonl 2>&1; done
for c in C4 C2 C1; do timeout 300 python bench.py --mode simulate --config $c --steps 3 --warmup 2 >> $out/simulate.jsonl 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c4_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $out/launches_c4_default.csv > $out/launches_c4_default.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:band_kernel -s 1 -c 1 -o /tmp/f_c4 -f python bench.py --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c4.log 2>&1
python tools/ncu_summary.py full /tmp/f_c4.ncu-rep > $out/ncu_full_c4.txt 2>&1; rm -f /tmp/f_c4.ncu-rep
timeout 900 ncu --set full --clock-control none -k regex:xband -s 1 -c 1 -o /tmp/f_c5 -f python bench.py --config C5 --frames 16384 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c5.log 2>&1
python tools/ncu_summary.py full /tmp/f_c5.ncu-rep > $out/ncu_full_c5.txt 2>&1; rm -f /tmp/f_c5.ncu-rep
