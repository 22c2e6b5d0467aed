mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c5_sampled or exchange or global_exchange" > gpurun_out/xt_tests.log 2>&1; echo EXIT $? >> gpurun_out/xt_tests.log
bash tools/ab_quick.sh xt "C5:8192 C5:16384" "xt||paper_2201_04265_b200/libldpc_b200.so" "xband2|LDPC_XTMEM=0|paper_2201_04265_b200/libldpc_b200.so"
