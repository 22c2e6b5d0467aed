bash tools/ab_quick.sh ab4 "C5:8192 C5:16384" "u32r||paper_2201_04265_b200/libldpc_b200.so" "adapt||build_ref/libldpc_r02_adapt.so"
bash tools/ab_quick.sh ab4 "C4:32768" "rpre2||paper_2201_04265_b200/libldpc_b200.so" "rpre1|LDPC_RPRE=1|paper_2201_04265_b200/libldpc_b200.so" "rpre0|LDPC_RPRE=0|paper_2201_04265_b200/libldpc_b200.so"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -q -m gpu -k "c5 or exchange or bench or auto" > gpurun_out/ab4_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab4_tests.log
