#!/bin/bash
# quick A/B: bench lines for a few workloads under several (env, lib) variants
# usage: bash tools/ab_quick.sh TAG "CFG:FRAMES ..." "LABEL|ENV|LIB" ...
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  IFS='|' read -r label envs lib <<< "$v"
  for c in $cfgs; do
    cfg=${c%%:*}; fr=${c##*:}
    extra=""; [ $cfg = C2 ] && extra="--ebn0 1.0"
    env $envs LDPC_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --frames $fr --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $extra 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$label', '$cfg', $fr, round(d['value'],3), 'Gbit/s sfu', round(r.get('sfu_model',r)['frac'],4), r['bound'], round(r['frac'],4), 'dec_ms', round(d['decode_ms_per_step'],3))
" >> gpurun_out/${tag}.log
  done
done
