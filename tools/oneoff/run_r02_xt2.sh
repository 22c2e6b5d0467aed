mkdir -p gpurun_out
timeout -s KILL 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -q -m gpu -x -k "c5 or exchange or global_exchange or three_slot or bench" > gpurun_out/xt2_tests.log 2>&1; echo EXIT $? >> gpurun_out/xt2_tests.log
bash tools/ab_quick.sh xt2 "C5:16384" "rtmem||paper_2201_04265_b200/libldpc_b200.so" "rws||build_ref/libldpc_r02_tmem2.so"
