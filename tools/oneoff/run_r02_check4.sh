mkdir -p gpurun_out
bash tools/ab_quick.sh t1 "T1-R3/4:1000 T1-R3/4:100000" "minb8||paper_2201_04265_b200/libldpc_b200.so" "head||build_ref/libldpc_r02_head.so"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "table_i or edge_kernel" > gpurun_out/t1_tests.log 2>&1; echo EXIT $? >> gpurun_out/t1_tests.log
