#!/bin/bash
# A/B: early-termination decided at the end of the variable phase (BAND_EDET, new lib) vs in the next check phase (old lib)
mkdir -p gpurun_out
for lib in ${LIBS:-paper_2201_04265_b200/libldpc_b200_edet1.so paper_2201_04265_b200/libldpc_b200.so}; do
  LDPC_LIB_PATH=$PWD/$lib timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        pts = d.get('sweep') or d.get('points') or []
        print('$lib', 'value', round(d['value'],4), 'dec_ms', round(d.get('decode_ms_per_step',0),4))
        for p in pts: print('   ', json.dumps(p)[:260])
" >> gpurun_out/edet_ab.log
done
