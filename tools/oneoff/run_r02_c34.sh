mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or explicit" > gpurun_out/c34_tests.log 2>&1; echo EXIT $? >> gpurun_out/c34_tests.log
bash tools/ab_quick.sh c34 "C3-R3/4:100000" "minb2||paper_2201_04265_b200/libldpc_b200.so" "minb3||build_ref/libldpc_r02_head3.so"
