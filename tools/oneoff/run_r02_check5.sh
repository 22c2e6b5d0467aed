mkdir -p gpurun_out
for lib in paper_2201_04265_b200/libldpc_b200.so build_ref/libldpc_r02_scalar.so; do
 for c in C2 C1 C3-R1/2 C4; do LDPC_LIB_PATH=$lib timeout 200 python bench.py --mode stream --config $c 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', '$c', round(d['value'],2), d['unit'], 'iters', round(d['mean_iterations'],2))
" >> gpurun_out/stream_ab.log; done; done
