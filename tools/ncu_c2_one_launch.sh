#!/bin/bash
# ncu evidence for C2's one-launch sweep: the launch list of the bench command
# and one --set full capture of the 50,000-frame decode launch.
out=gpurun_out/s5; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c2.csv \
  python bench.py --config C2 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c2_launch.log 2>&1
python tools/ncu_summary.py launches $out/launches_c2.csv > $out/launches_c2.txt 2>&1
# --eager --steps 1 --warmup 1: every point decodes 3 times (plan, warm-up, timed), then the one-launch batch 3
# times: band_kernel launches 15-17 are the 50,000-frame ones; capture the timed one (index 17)
timeout 900 ncu --set full --clock-control none -k regex:band_kernel -s 17 -c 1 -o /tmp/f_c2one -f \
  python bench.py --config C2 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c2_full.log 2>&1
python tools/ncu_summary.py full /tmp/f_c2one.ncu-rep > $out/ncu_full_c2_one_launch.txt 2>&1; rm -f /tmp/f_c2one.ncu-rep
tail -30 $out/launches_c2.txt; head -30 $out/ncu_full_c2_one_launch.txt
