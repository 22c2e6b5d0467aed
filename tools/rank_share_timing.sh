#!/bin/bash
# One rank's share of a strong-scaling step at N = 1, 2, 4, 8, timed on one GPU
# (the ranks share nothing but a 48-byte counter all-reduce, so a rank's step is
# its own work): C4's 200,000 frames and C5's 10^6 frames split by Eq. 9.
out=gpurun_out/s5/rank_share.txt; mkdir -p gpurun_out/s5; rm -f $out
run() {  # config total N
  fr=$(( ($2 + $3 - 1) / $3 ))
  timeout 900 python bench.py --config $1 --frames $fr --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$1 N=$3 rank share', $fr, 'frames: step', round(d['ms_per_step'], 3), 'ms, decode', round(d['decode_ms_per_step'], 3), 'ms,', round(d['value'], 4), 'Gbit/s per GPU, SFU frac', round(d['roofline'].get('sfu_model', d['roofline'])['frac'], 4))
" >> $out
}
for N in 1 2 4 8; do run C4 200000 $N; done
for N in 8 4; do run C5 1000000 $N; done
cat $out
