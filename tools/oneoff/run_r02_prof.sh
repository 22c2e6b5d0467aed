# r02 profiling call: microbenchmarks (cluster placement, LOP3/POPC), issue
# profiles of every workload's decode launch, ncu --set full of the C4 encode.
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK | head -30 > gpurun_out/p_clocks.txt
./tools/microbench_cluster > gpurun_out/p_cluster.txt 2>&1
./tools/microbench_lop > gpurun_out/p_lop.txt 2>&1
timeout 2400 python tools/issue_profile.py gpurun_out/issue.json > gpurun_out/p_issue.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_parity -c 1 -o gpurun_out/enc_c4 -f python bench.py --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/p_enc.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/p_c4.log 2>&1
