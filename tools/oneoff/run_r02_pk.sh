mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c2 or c3 or c4 or simulate or explicit or table or c1" > gpurun_out/pk_tests.log 2>&1; echo EXIT $? >> gpurun_out/pk_tests.log
bash tools/ab_quick.sh pk "C1:1000 C2:10000 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:200000 T1-R1/4:1000 T1-R3/4:1000" "pk||paper_2201_04265_b200/libldpc_b200.so"
