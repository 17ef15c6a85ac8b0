P2S_BENCH_DEBUG=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra 2>&1 | tail -4 | cut -c1-600
