for i in 1 2 3; do
for m in blur render; do
P2S_FUSED_LOOP=$m python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$m', 'step', round(d['ms_per_step']*1e3,1), 'fused', round(r['fused_ms_median']*1e3,1), 'min', round(r['fused_ms_min']*1e3,1), 'max', round(r['fused_ms_max']*1e3,1), 'evented', round(r['evented_render_ms_median']*1e3,1), d['clocks']['all_legs']['reasons'])"
done
done
