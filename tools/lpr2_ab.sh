#!/bin/bash
# Lane-pair band kernel (LPR = 2) check: targeted GPU tests, then the
# small-batch configs with and without it (LDPC_NO_LPR2=1).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "c1 or table_i or simulate or auto or edge or explicit or no_exemptions or trees or deterministic" > gpurun_out/lpr2_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/lpr2_tests.log
for c in C1:1000 T1-R1/4:1000 T1-R1/2:1000 T1-R3/4:1000; do
  cfg=${c%%:*}; fr=${c##*:}
  timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline 2>&1 | grep "^{" >> gpurun_out/lpr2_bench.log
  LDPC_NO_LPR2=1 timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline 2>&1 | grep "^{" >> gpurun_out/lpr2_bench_base.log
done
for c in C1 T1-R3/4; do LDPC_NO_EDGE=1 timeout 120 python bench.py --mode stream --config $c 2>&1 | grep "^{" >> gpurun_out/lpr2_stream.log; done
