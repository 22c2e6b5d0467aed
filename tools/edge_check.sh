#!/bin/bash
# Lane-per-edge kernel (variant 8) check: the GPU test suite and stream mode of
# the small configs against the band kernel (LDPC_NO_EDGE=1).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/edge_tests3.log 2>&1; echo "EXIT $?" >> gpurun_out/edge_tests3.log
for c in C1 T1-R1/4 T1-R1/2 T1-R3/4 C2; do
  timeout 120 python bench.py --mode stream --config $c >> gpurun_out/edge_stream3.log 2>&1
  LDPC_NO_EDGE=1 timeout 120 python bench.py --mode stream --config $c >> gpurun_out/edge_stream3_base.log 2>&1
done
