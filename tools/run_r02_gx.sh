mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c5_sampled and 9" > gpurun_out/gx_tests.log 2>&1; echo EXIT $? >> gpurun_out/gx_tests.log
grep -q "EXIT 0" gpurun_out/gx_tests.log || exit 0
bash tools/ab_quick.sh gx "C5:8192 C5:16384" "gx|LDPC_GX=1|paper_2201_04265_b200/libldpc_b200.so" "xband2||paper_2201_04265_b200/libldpc_b200.so"
