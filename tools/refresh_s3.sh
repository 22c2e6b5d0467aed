#!/bin/bash
# Final round-2 refresh after the small-batch / count-kernel changes: GPU
# tests, smoke, one bench line per workload, the default bench line, the C2
# sweep, all 10^6 C5 frames, the reference arm, stream and simulate modes,
# torchrun N = 1, the C4 launch list and an ncu --set full capture of the
# C4 decode launch.
out=gpurun_out/s3; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "EXIT $?" >> $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "EXIT $?" >> $out/smoke.log
bash tools/bench_all.sh $out/all_configs.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_default.jsonl 2>&1
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_c2_sweep.jsonl 2>&1
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_c5_full.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.jsonl 2>&1
for c in C1 T1-R1/4 T1-R1/2 T1-R3/4 C2 C3-R1/2 C4 C5; do timeout 200 python bench.py --mode stream --config $c >> $out/stream.jsonl 2>&1; done
for c in C4 C2 C1; do timeout 300 python bench.py --mode simulate --config $c --steps 3 --warmup 3 >> $out/simulate.jsonl 2>&1; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > $out/torchrun_n1.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c4_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $out/launches_c4_default.csv > $out/launches_c4_default.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:band_kernel -s 1 -c 1 -o /tmp/f_c4 -f python bench.py --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $out/ncu_c4.log 2>&1
python tools/ncu_summary.py full /tmp/f_c4.ncu-rep > $out/ncu_full_c4.txt 2>&1; rm -f /tmp/f_c4.ncu-rep
