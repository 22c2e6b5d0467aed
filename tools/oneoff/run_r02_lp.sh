mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "table or lane_pair" > gpurun_out/lp_tests.log 2>&1; echo EXIT $? >> gpurun_out/lp_tests.log
bash tools/ab_quick.sh lp "T1-R1/4:1000 T1-R1/2:1000 T1-R1/4:100000 T1-R1/2:100000" "minb4||paper_2201_04265_b200/libldpc_b200.so" "minb5||build_ref/libldpc_r02_head3.so"
