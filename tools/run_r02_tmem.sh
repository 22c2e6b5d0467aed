mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c4 or explicit or auto or simulate" > gpurun_out/tmem_tests.log 2>&1; echo EXIT $? >> gpurun_out/tmem_tests.log
bash tools/ab_quick.sh tmem "C4:200000 C4:32768" "tmem||paper_2201_04265_b200/libldpc_b200.so" "head||build_ref/libldpc_r02_head.so"
