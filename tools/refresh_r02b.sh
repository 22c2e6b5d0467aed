#!/bin/bash
# Round-2 refresh after the tensor-core encoder and the C5 idle-SM groups:
# GPU tests, the default bench line, every config, the C2 sweep, the reference
# arm, the launch list of the default bench and a torchrun (N = 1) pass.
out=gpurun_out/refresh; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gputest.log 2>&1; tail -3 $out/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_default.jsonl 2>&1
bash tools/bench_all.sh $out/all_configs.jsonl
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_c2_sweep.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c4_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $out/launches_c4_default.csv > $out/launches_c4_default.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $out/torchrun_c4.jsonl 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 1 --config C5 --frames 65536 --steps 3 --warmup 3 --no-cpu-baseline > $out/torchrun_c5.jsonl 2>&1
grep -h '^{' $out/bench_default.jsonl $out/torchrun_c4.jsonl $out/torchrun_c5.jsonl | cut -c1-300
