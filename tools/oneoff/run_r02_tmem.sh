mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c4 or explicit or auto or simulate" > gpurun_out/tmem2_tests.log 2>&1; echo EXIT $? >> gpurun_out/tmem2_tests.log
bash tools/ab_quick.sh tmem2 "C4:200000" "tmem2||paper_2201_04265_b200/libldpc_b200.so" "tmem1||build_ref/libldpc_r02_tmem1.so"
