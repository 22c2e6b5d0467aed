mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1 or simulate or no_exemptions" > gpurun_out/c1_tests.log 2>&1; echo EXIT $? >> gpurun_out/c1_tests.log
bash tools/ab_quick.sh c1i "C1:1000" "c1i||paper_2201_04265_b200/libldpc_b200.so" "head3||build_ref/libldpc_r02_head3.so"
