mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/full2_tests.log 2>&1; echo EXIT $? >> gpurun_out/full2_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/full2_bench.log 2>&1
