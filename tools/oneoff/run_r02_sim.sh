mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "simulate" > gpurun_out/sim_tests.log 2>&1; echo EXIT $? >> gpurun_out/sim_tests.log
timeout 300 python bench.py --mode simulate --config C4 --steps 3 --warmup 2 > gpurun_out/sim_c4.log 2>&1
