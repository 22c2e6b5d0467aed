#!/bin/bash
# C2's sweep as one launch: points by ascending Eb/N0 (longest-running frames
# first, the default) against descending, twice each on one box.
out=gpurun_out/s5; mkdir -p $out; rm -f $out/c2_order_ab.txt
for o in asc desc asc desc; do
  timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --sweep-order $o 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); o = d['sweep_one_launch']
        print('order', o['order_ebn0_db'], 'points one by one', round(d['value'], 3), 'Gbit/s; one launch', round(o['value'], 3),
              'Gbit/s, decode', round(o['decode_ms_per_step'], 3), 'ms, frac', round(o['roofline_frac_on_executed_iterations'], 3),
              'counters match', o['counters_match_points'])
" >> $out/c2_order_ab.txt
done
cat $out/c2_order_ab.txt
