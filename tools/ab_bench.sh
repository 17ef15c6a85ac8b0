# A/B the fused kernel of two library builds in one session (alternating, 3 rounds)
for round in 1 2 3; do
  for v in A B; do
    P2S_LIB=paper_2107_11627_b200/libp2s_$v.so timeout 300 python bench.py --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v round $round', round(d['value'],1), 'fps fused mean', round(r['fused_ms_mean']*1e3,1), 'min', round(r['fused_ms_min']*1e3,1), 'us frac', round(r['frac'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'])"
  done
done
