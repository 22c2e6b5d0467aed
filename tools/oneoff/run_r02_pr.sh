mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c2 or table or explicit or early or simulate or no_exemptions" > gpurun_out/pr_tests.log 2>&1; echo EXIT $? >> gpurun_out/pr_tests.log
bash tools/ab_quick.sh pr "C2:10000 T1-R3/4:1000 T1-R3/4:100000" "pr||paper_2201_04265_b200/libldpc_b200.so" "head3||build_ref/libldpc_r02_head3.so"
for lib in paper_2201_04265_b200/libldpc_b200.so build_ref/libldpc_r02_head3.so; do LDPC_LIB_PATH=$lib timeout 300 python bench.py --config C2 --ebn0 3.0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$lib C2@3dB', round(d['value'],3), round(d['roofline']['frac'],4))" >> gpurun_out/pr.log; done
