bash tools/ab_quick.sh ab3 "C5:8192 C5:16384" "ns3||paper_2201_04265_b200/libldpc_b200.so" "ns2|LDPC_XBAND_SLOTS=2|paper_2201_04265_b200/libldpc_b200.so" "adapt||build_ref/libldpc_r02_adapt.so"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c5 or exchange" > gpurun_out/ab3_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab3_tests.log
