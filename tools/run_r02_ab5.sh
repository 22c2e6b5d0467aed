bash tools/ab_quick.sh ab5 "T1-R3/4:1000 T1-R3/4:100000" "lpr1||paper_2201_04265_b200/libldpc_b200.so" "lpr2|LDPC_LPR2_ALL=1|paper_2201_04265_b200/libldpc_b200.so"
bash tools/ab_quick.sh ab5 "C4:200000" "c4||paper_2201_04265_b200/libldpc_b200.so"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "table_i or c4 or lane_pair" > gpurun_out/ab5_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab5_tests.log
LDPC_LPR2_ALL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "table_i" > gpurun_out/ab5_tests_lpr2.log 2>&1; echo EXIT $? >> gpurun_out/ab5_tests_lpr2.log
