#!/bin/bash
# Stream-mode latency of the exchange cluster kernel by cluster size
# (LDPC_XBAND_C, fixed at bind time).  Usage: bash tools/xc_sweep.sh
mkdir -p gpurun_out
for C in 4 5 6 9 10 12 15; do
  echo "C=$C" >> gpurun_out/xc_sweep.log
  LDPC_XBAND_C=$C timeout 120 python bench.py --mode stream --config C4 2>&1 | grep "^{" >> gpurun_out/xc_sweep.log
done
for C in 2 3 6 9; do
  echo "C=$C" >> gpurun_out/xc_sweep.log
  LDPC_XBAND_C=$C timeout 120 python bench.py --mode stream --config C3-R1/2 2>&1 | grep "^{" >> gpurun_out/xc_sweep.log
done
