for i in 1 2; do for r in 0.50 0.53 0.56; do
LDPC_XTAIL_RATE=$r timeout 600 python bench.py --config C5 --frames 131072 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$r', round(d['value'],4), round(d['roofline']['frac'],4), round(d['decode_ms_per_step'],2))"
done; done
