mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c2 or c3 or c4 or simulate or explicit or early or count" > gpurun_out/av_tests.log 2>&1; echo EXIT $? >> gpurun_out/av_tests.log
bash tools/ab_quick.sh av "C2:10000 C3-R1/4:100000 C3-R1/2:100000 C3-R3/4:100000 C4:200000" "adapt||paper_2201_04265_b200/libldpc_b200.so" "always||build_ref/libldpc_r02_rtmem.so"
for lib in paper_2201_04265_b200/libldpc_b200.so build_ref/libldpc_r02_rtmem.so; do LDPC_LIB_PATH=$lib timeout 300 python bench.py --config C2 --ebn0 3.0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$lib C2@3dB', round(d['value'],3), round(d['roofline']['frac'],4), 'iters', d['mean_iterations'])" >> gpurun_out/av.log; done
