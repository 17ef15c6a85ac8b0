for P in 0 1; do
  echo "== progressive=$P"
  P2S_PROGRESSIVE=$P P2S_LIB=paper_2107_11627_b200/libp2s_prof.so timeout 120 python tools/role_profile.py 3 2>&1 | tail -18
  P2S_PROGRESSIVE=$P timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_p$P.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_p$P.log').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['fused_ms_mean'], d['roofline']['frac'])"
done
