for lib in paper_2201_04265_b200/libldpc_b200.so build_ref/libldpc_r02_adapt.so; do
  LDPC_LIB_PATH=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); e=d['encode_roofline']
        print('$lib', round(d['value'],4), 'Gbit/s', 'decode', round(d['roofline']['frac'],4), 'encode_ms', round(e['ms_per_step'],3), 'encode_frac', round(e['frac'],4))
" >> gpurun_out/ab6.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "encode or simulate or count" > gpurun_out/ab6_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab6_tests.log
