#!/bin/bash
# One GPU call: GPU tests, smoke, the default bench line, every config's bench
# line, stream and simulate modes.  Usage: bash tools/gpu_round_check.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke_$tag.log
timeout 400 python bench.py > gpurun_out/bench_default_$tag.log 2>&1
bash tools/bench_all.sh gpurun_out/cfg_$tag.log
for c in C1 C3-R1/2 C4 C5; do timeout 120 python bench.py --mode stream --config $c >> gpurun_out/stream_$tag.log 2>&1; done
for c in C4 C2; do timeout 300 python bench.py --mode simulate --config $c --steps 3 --warmup 2 >> gpurun_out/simulate_$tag.log 2>&1; done
