cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -k "color" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/t.log
for v in 0 1 0 1; do
if [ $v = 1 ]; then export P2S_COLOR_FUSED=1; else unset P2S_COLOR_FUSED; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-configs --no-anchor-mode --no-batch-mode --no-adjoint-mode --no-sequence-mode > gpurun_out/col_$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/col_$v.log').read().strip().splitlines()[-1])
print('COLOR_FUSED=$v', round(d['color_mode']['value']), round(d['color_mode'].get('adjoint_value', 0)))"
done
