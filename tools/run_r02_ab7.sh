bash tools/ab_quick.sh ab7 "C4:32768 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000" "pfo||paper_2201_04265_b200/libldpc_b200.so" "enc||build_ref/libldpc_r02_enc.so"
