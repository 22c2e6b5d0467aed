mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bench.py -q -m gpu > gpurun_out/c3_tests.log 2>&1; echo EXIT $? >> gpurun_out/c3_tests.log
for c in C1:1000 T1-R3/4:1000 C4:200000; do cfg=${c%%:*}; fr=${c##*:}; timeout 300 python bench.py --config $cfg --frames $fr --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3_$cfg.log 2>&1; done
