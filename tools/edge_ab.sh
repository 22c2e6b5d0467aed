mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "edge or c1_batch or table_i or simulate_equals or irregular or trees or auto or edge_cases or no_exemptions" > gpurun_out/edge_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/edge_tests.log
for c in C1:1000 T1-R1/4:1000 T1-R1/2:1000 T1-R3/4:1000; do
  cfg=${c%%:*}; fr=${c##*:}
  timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline >> gpurun_out/edge_ab.log 2>&1
  LDPC_NO_EDGE=1 timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline >> gpurun_out/edge_ab_base.log 2>&1
  LDPC_EDGE_NOVOTE=1 timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline >> gpurun_out/edge_ab_novote.log 2>&1
done
for c in C1 T1-R1/2; do timeout 120 python bench.py --mode stream --config $c >> gpurun_out/edge_stream.log 2>&1; LDPC_NO_EDGE=1 timeout 120 python bench.py --mode stream --config $c >> gpurun_out/edge_stream_base.log 2>&1; done
