mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c4 or simulate or auto" > gpurun_out/t6_tests.log 2>&1; echo EXIT $? >> gpurun_out/t6_tests.log
bash tools/ab_quick.sh t6 "C4:200000" "t6||paper_2201_04265_b200/libldpc_b200.so" "head2||build_ref/libldpc_r02_head2.so"
