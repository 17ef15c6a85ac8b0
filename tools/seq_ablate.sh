# Timing-only ablations of sequence mode (50 frames of one cfg3 image; results WRONG by construction)
# build: bash tools/seq_ablate.sh build ; run on the GPU: bash tools/seq_ablate.sh run
set -e
cd "$(dirname "$0")/.."
V="base: NODRAIN:-DP2S_ABL_NODRAIN NOA2:-DP2S_ABL_NOA2 EPI0:-DP2S_ABL_EPI0 NOMLPMMA:-DP2S_ABL_NOMLPMMA"
if [ "$1" = build ]; then
  for v in $V; do
    n=${v%%:*}; f=${v#*:}
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -maxrregcount=144 -Iinclude -Ipaper_2107_11627_b200/csrc $f \
      paper_2107_11627_b200/csrc/p2s_host.cu paper_2107_11627_b200/csrc/p2s_sampler.cu \
      paper_2107_11627_b200/csrc/p2s_anchor.cu -o paper_2107_11627_b200/abl_$n.so &
  done
  wait
else
  for v in $V; do
    n=${v%%:*}
    P2S_LIB=paper_2107_11627_b200/abl_$n.so timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
      --no-configs --no-anchor-mode --no-batch-mode --no-adjoint-mode > gpurun_out/sabl_$n.log 2>&1 || true
    python -c "
import json; d=json.loads(open('gpurun_out/sabl_$n.log').read().strip().splitlines()[-1]); print('$n', 'render', round(d['value']), 'seq', round(d['sequence_mode']['value']), 'color', round(d['color_mode']['value']))" || tail -3 gpurun_out/sabl_$n.log
  done
fi
