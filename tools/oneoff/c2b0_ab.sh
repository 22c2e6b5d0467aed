#!/bin/bash
# C2 A/B: one band-0 row per thread at 7 CTAs/SM (default) vs two rows per thread at 12 / 14 CTAs/SM (LDPC_C2_B0=2)
mkdir -p gpurun_out
run() {
  label=$1; shift
  env "$@" timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print('$label', 'value', round(d['value'],4), ' '.join(f\"{p['ebn0_db']}:{p['decode_ms_per_step']:.4f}\" for p in d['points']))
" >> gpurun_out/c2b0_ab.log
}
for i in 1 2; do
  run b0_1
  run b0_2_m12 LDPC_C2_B0=2
  run b0_2_m14 LDPC_C2_B0=2 LDPC_LIB_PATH=$PWD/paper_2201_04265_b200/libldpc_b200_c2m14.so
done
