# one GPU call: parity (quick subset), role profile, bench line summary
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -2
P2S_LIB=paper_2107_11627_b200/libp2s_prof.so timeout 120 python -u tools/role_profile.py ${CFG:-3} 2>&1 | tail -18
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print('BENCH', round(d['value'],1), 'fps', round(d['roofline']['fused_ms_mean']*1e3,1), 'us fused', round(d['ms_per_step']*1e3,1), 'us step', round(d['roofline']['clean_step_ms']*1e3,1), 'clean', round(d['roofline']['frac'],4), d['clocks'])"
