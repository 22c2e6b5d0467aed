#!/bin/bash
# A/B of two library builds (gpurun_lib_base.so vs gpurun_lib_minb.so, built
# locally with different launch bounds) on the configs they affect.
mkdir -p gpurun_out
for v in base minb base minb; do
  cp gpurun_lib_$v.so paper_2201_04265_b200/libldpc_b200.so
  for c in T1-R3/4:1000 T1-R3/4:100000; do
    cfg=${c%%:*}; fr=${c##*:}
    echo "== $v $cfg $fr" >> gpurun_out/minb3_ab.log
    timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline 2>&1 | grep "^{" >> gpurun_out/minb3_ab.log
  done
done
