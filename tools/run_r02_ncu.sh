# r02: full ncu captures of the decode launch for C2 (1.0 dB, 10k frames), C3-R1/2, C5 (one chunk), C4; FFMA2 microbench
mkdir -p gpurun_out
./tools/microbench_ffma2 > gpurun_out/p_ffma2.txt 2>&1
K="regex:band_kernel|xband"
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o gpurun_out/ncu_c2 -f python bench.py --config C2 --ebn0 1.0 --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o gpurun_out/ncu_c5 -f python bench.py --config C5 --frames 16384 --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o gpurun_out/ncu_c3r12 -f python bench.py --config C3-R1/2 --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3r12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o gpurun_out/ncu_c4 -f python bench.py --frames 32768 --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1
