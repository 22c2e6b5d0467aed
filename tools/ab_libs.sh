#!/bin/bash
# A/B of two library builds on one GPU box: bit-for-bit output comparison
# (tools/compare_libs.py) and one bench line per workload for each build.
# Usage: bash tools/ab_libs.sh OLD.so NEW.so TAG
old=$1; new=$2; tag=${3:-ab}
mkdir -p gpurun_out
python tools/compare_libs.py run --lib $old --out gpurun_out/${tag}_old.npz > gpurun_out/${tag}_cmp.log 2>&1
python tools/compare_libs.py run --lib $new --out gpurun_out/${tag}_new.npz >> gpurun_out/${tag}_cmp.log 2>&1
python tools/compare_libs.py diff gpurun_out/${tag}_old.npz gpurun_out/${tag}_new.npz >> gpurun_out/${tag}_cmp.log 2>&1
rm -f gpurun_out/${tag}_old.npz gpurun_out/${tag}_new.npz
for lib in $new $old; do
  for c in C1:1000 C2:10000 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:16384 C5:8192 T1-R1/4:1000 T1-R1/2:1000 T1-R3/4:1000; do
    cfg=${c%%:*}; fr=${c##*:}
    extra=""; [ $cfg = C2 ] && extra="--ebn0 1.0"
    LDPC_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --frames $fr --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $extra 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$lib', '$cfg', $fr, round(d['value'],3), 'Gbit/s', round(r.get('sfu_model',r)['frac'],4), r['bound'], round(r['frac'],4))
" >> gpurun_out/${tag}_bench.log
  done
done
