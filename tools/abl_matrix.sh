for n in base notma nomlp epi0 noe nodrain nosimt nosimt_notma noconv base; do
  P2S_LIB=paper_2107_11627_b200/abl_$n.so timeout 90 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/abl_$n.log 2>&1
  rc=$?
  python - "$n" "$rc" <<'P'
import json, sys
n, rc = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/abl_{n}.log").read().strip().splitlines()[-1])
    print(n, "rc", rc, round(d["roofline"]["fused_ms_median"] * 1e3, 1), "us fused;", round(d["ms_per_step"] * 1e3, 1), "us step")
except Exception as e:
    print(n, "rc", rc, "no result")
P
done
