# Timing-only ablations of k_fused_p2s (results are WRONG by construction; never used for parity).
# Build locally:   bash tools/ablate.sh build      -> paper_2107_11627_b200/abl_*.so
# Run on the GPU:  bash tools/ablate.sh run
set -e
cd "$(dirname "$0")/.."
V="${ABL_V:-base: MMA2:-DP2S_MMA_WARP2}"
if [ "$1" = build ]; then
  for v in $V; do
    n=${v%%:*}; f=${v#*:}; f=${f//_-D/ -D}
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -maxrregcount=144 -Iinclude -Ipaper_2107_11627_b200/csrc $f \
      paper_2107_11627_b200/csrc/p2s_host.cu paper_2107_11627_b200/csrc/p2s_sampler.cu paper_2107_11627_b200/csrc/p2s_anchor.cu \
      -o paper_2107_11627_b200/abl_$n.so &
  done
  wait
else
  for v in $V; do
    n=${v%%:*}
    P2S_LIB=paper_2107_11627_b200/abl_$n.so timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abl_$n.log 2>&1 || true
    python -c "
import json,sys; d=json.loads(open('gpurun_out/abl_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['roofline']['fused_ms_mean']*1e3,1), 'us')" || tail -3 gpurun_out/abl_$n.log
  done
fi
