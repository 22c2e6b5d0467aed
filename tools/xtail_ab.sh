#!/bin/bash
# C5 A/B: exchange clusters alone vs clusters + global-exchange tail on the idle SMs
mkdir -p gpurun_out
out=gpurun_out/xtail_ab.log
run() {
  label=$1; shift
  env "$@" timeout 600 python bench.py --config C5 --frames 65536 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$label', round(d['value'],4), 'Gbit/s sfu', round(r.get('sfu_model',r)['frac'],4), 'dec_ms', round(d['decode_ms_per_step'],3))
" >> $out
}
run notail LDPC_XTAIL=0
run tail055 LDPC_XTAIL_RATE=0.55
run tail045 LDPC_XTAIL_RATE=0.45
run tail065 LDPC_XTAIL_RATE=0.65
run tail080 LDPC_XTAIL_RATE=0.80
