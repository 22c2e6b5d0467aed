for e in 3.0 2.0; do for f in 10000 40000 160000; do
timeout 300 python bench.py --config C2 --ebn0 $e --frames $f --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$e', $f, 'dec_ms', round(d['decode_ms_per_step'],4), 'iters', round(d['mean_iterations'],3), 'frac', round(d['roofline']['frac'],4))
" >> gpurun_out/tail.log
done; done
