set -x
timeout 900 python -m pytest tests/test_gpu_bench.py tests/test_gpu_parity.py -m gpu -q -rf -k "bench or irregular or simulate or alist" > gpurun_out/t2.log 2>&1; echo EXIT $? >> gpurun_out/t2.log
timeout 300 python -m pytest tests/test_gpu_psi.py -q -s > gpurun_out/t2_psi.log 2>&1; echo EXIT $? >> gpurun_out/t2_psi.log
timeout 400 python bench.py --steps 3 --warmup 3 > gpurun_out/b2_c4.log 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b2_c2.log 2>&1
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b2_c5.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b2_ref.log 2>&1
