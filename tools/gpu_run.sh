python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['configs']
for k,v in c.items(): print(k, round(v['value']), round(v['roofline']['frac'],3), v.get('batched') and (round(v['batched']['value']), round(v['batched']['roofline']['frac'],3)))"
