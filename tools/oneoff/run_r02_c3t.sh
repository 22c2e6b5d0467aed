mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or c4 or explicit or simulate" > gpurun_out/c3t_tests.log 2>&1; echo EXIT $? >> gpurun_out/c3t_tests.log
bash tools/ab_quick.sh c3t "C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:200000" "c3t||paper_2201_04265_b200/libldpc_b200.so"
