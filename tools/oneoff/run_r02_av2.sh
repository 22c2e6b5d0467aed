mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c2 or c3 or c4 or simulate or explicit or early or count or table" > gpurun_out/av2_tests.log 2>&1; echo EXIT $? >> gpurun_out/av2_tests.log
bash tools/ab_quick.sh av2 "C2:10000 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:200000 T1-R3/4:100000" "sel||paper_2201_04265_b200/libldpc_b200.so"
