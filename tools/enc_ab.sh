#!/bin/bash
# encoder A/B: tensor-core parity product vs the INT-pipe binary GEMM, warp-per-frame vs CTA-per-frame assemble
mkdir -p gpurun_out
for cfg in "C4 200000" "C3-R1/2 100000" "C5 65536"; do
  set -- $cfg
  for v in "mma_warp|" "mma_cta|LDPC_ASM_WARP=0" "int_cta|LDPC_ENC_MMA=0 LDPC_ASM_WARP=0"; do
    IFS='|' read -r label envs <<< "$v"
    env $envs timeout 900 python bench.py --config $1 --frames $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); e=d.get('encode_roofline') or {}
        print('$1', '$label', round(d['value'],4), 'Gbit/s step_ms', round(d['ms_per_step'],3), 'dec_ms', round(d['decode_ms_per_step'],3), 'enc_ms', round(e.get('ms_per_step',0),3), e.get('bound'), 'enc_frac', round(e.get('frac',0),3))
" >> gpurun_out/enc_ab2.log
  done
done
