for lib in paper_2107_11627_b200/libp2s.so paper_2107_11627_b200/abl_seq.so; do
P2S_LIB=$lib python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-configs --no-anchor-mode --no-batch-mode --no-adjoint-mode 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', 'render', round(d['value']), 'seq', round(d['sequence_mode']['value']), 'color', round(d['color_mode']['value']))" || true
done
