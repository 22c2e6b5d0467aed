mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/c2_tests.log 2>&1; echo EXIT $? >> gpurun_out/c2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2_smoke.log 2>&1; echo EXIT $? >> gpurun_out/c2_smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/c2_torchrun.log 2>&1; echo EXIT $? >> gpurun_out/c2_torchrun.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/c2_torchrun_ref.log 2>&1; echo EXIT $? >> gpurun_out/c2_torchrun_ref.log
