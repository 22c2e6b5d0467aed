#!/bin/bash
# ncu evidence for the round-2 plan changes: issue profile of C2 and C3-R1/2
# (merged into profiles/issue.json) and --set full captures of their decode launches
out=gpurun_out/ncu_r02c; mkdir -p $out
cp profiles/issue.json $out/issue.json
timeout 1500 python tools/issue_profile.py $out/issue.json C2,C3-R1/2 > $out/issue.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:band_kernel -s 1 -c 1 -o $out/c2 -f python bench.py --config C2 --ebn0 1.0 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c2.log 2>&1
python tools/ncu_summary.py full $out/c2.ncu-rep > $out/ncu_full_c2.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:band_kernel -s 1 -c 1 -o $out/c3 -f python bench.py --config C3-R1/2 --frames 100000 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c3.log 2>&1
python tools/ncu_summary.py full $out/c3.ncu-rep > $out/ncu_full_c3r12.txt 2>&1
rm -f $out/*.ncu-rep
cat $out/issue.log; head -30 $out/ncu_full_c2.txt; head -30 $out/ncu_full_c3r12.txt
