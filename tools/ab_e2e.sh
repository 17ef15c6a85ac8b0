# A/B of the e2e leg (p2s_render_host) between two builds on one box: build the baseline into
# paper_2107_11627_b200/libp2s_old.so first (same nvcc flags as build.py), then run this via gpurun.
for i in 1 2 3 4; do
for lib in libp2s_old.so libp2s.so; do
P2S_LIB=$PWD/paper_2107_11627_b200/$lib python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --e2e-steps 150 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['e2e']['value'],1))"
done; done
