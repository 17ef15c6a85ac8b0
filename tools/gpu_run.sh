cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "sequence or color or graph" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/t.log
for v in 0 1 0 1; do
if [ $v = 1 ]; then export P2S_NO_L1EARLY=1; else unset P2S_NO_L1EARLY; fi
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode --no-adjoint-mode --no-configs --no-batch-mode > gpurun_out/sq_$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/sq_$v.log').read().strip().splitlines()[-1])
print('NO_L1EARLY=$v', round(d['value']), 'seq', round(d['sequence_mode']['value']), 'col', round(d['color_mode']['value']))"
done
