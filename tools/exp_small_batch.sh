#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/exp1.log
for c in "T1-R1/4" "T1-R1/2" "T1-R3/4" "C1"; do
 for fr in 1000 740 592 444 296 260 148; do
  for v in 0 8; do
   timeout 120 python bench.py --config $c --frames $fr --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --variant $v 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$c', $fr, 'v$v', round(d['value'],3), 'Gbit/s sfu', round(r.get('sfu_model',r)['frac'],4), 'dec_ms', round(d['decode_ms_per_step'],4), 'step_ms', round(d['ms_per_step'],4))
" >> $out
  done
 done
done
