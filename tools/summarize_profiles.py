"""Summarise gpurun_out/ ncu captures into profiles/ (committed evidence).

  python tools/summarize_profiles.py <round-tag>
Writes profiles/<tag>_launches.csv (per-launch device times of one bench invocation),
profiles/<tag>_launch_shares.txt, profiles/<tag>_ncu_fused.txt (key metrics of one
--set full capture of k_fused_p2s) and profiles/ncu_fused_summary.json (read by bench.py:
DRAM bytes per launch for roofline.traffic).
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

# ---- launch list
rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    name = r[ki].split("(")[0].split("<")[0].removeprefix("void ")  # (template instantiations folded)
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
ours = {k: v for k, v in tot.items() if k.startswith("p2s::")}
# one render = one launch of each of our kernels (the bench's dedicated fused-kernel loop adds
# fused launches without a warp, so shares use per-launch averages)
step_ns = sum(v / cnt[k] for k, v in ours.items())
with open(os.path.join(PROF, f"{tag}_launch_shares.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    f.write("of: python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e\n\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"{tot[k] / cnt[k] / 1e3:10.1f} us/launch x{cnt[k]:3d}  {k}\n")
    f.write("\nshare of one p2s_render (our kernels only):\n")
    for k, v in ours.items():
        f.write(f"  {k:28s} {v / cnt[k] / step_ns * 100:5.1f} %  (per-launch average / sum of averages)\n")

# ---- full capture of the fused kernel
rep = os.path.join(OUT, "prof_fused.ncu-rep")
if not os.path.exists(rep):  # a launch-list-only evidence run (tools/evidence_run.sh): keep the last capture
    print(open(os.path.join(PROF, f"{tag}_launch_shares.txt")).read())
    sys.exit(0)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, v = rr[0], rr[1], rr[2]
m = {a: (c, b) for a, b, c in zip(h, u, v)}
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum",
        "smsp__mem_tensor_writes_op_utcmma.sum", "launch__shared_mem_per_block_dynamic"]
lines = []
for k in want:
    if k in m:
        lines.append(f"{k:80s} {m[k][0]:>16s} {m[k][1]}")


def to_bytes(val, unit):
    val = float(val.replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
with open(os.path.join(PROF, f"{tag}_ncu_fused.txt"), "w") as f:
    f.write("ncu --set full --clock-control none -k regex:k_fused -s 1 -c 1 (cfg3, one frame)\n\n")
    f.write("\n".join(lines) + "\n")
    f.write(f"\nDRAM bytes per launch (read+write): {dram:.0f}\n")
def num(k):
    return float(m[k][0].replace(",", "")) if k in m else None


clk = num("sm__cycles_elapsed.avg.per_second")  # the capture's own clock record (GHz)
json.dump({"dram_bytes_per_launch": dram, "source": f"profiles/{tag}_ncu_fused.txt",
           "kernel": "k_fused_p2s", "workload": "cfg3_512_rgb_K100_S33",
           "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
           "tc_smem_pipe_pct": num("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
           "sm_clock_ghz": clk, "gpu_time_us": num("gpu__time_duration.sum"),
           "note": "ncu --set full --clock-control none (replayed ~40x); sm_clock_ghz = sm__cycles_elapsed."
                   "avg.per_second of the capture: the tensor-pipe % is a fraction of elapsed cycles at that "
                   "clock, the duration is not comparable to bench timings at a different clock"},
          open(os.path.join(PROF, "ncu_fused_summary.json"), "w"), indent=1)
print(open(os.path.join(PROF, f"{tag}_launch_shares.txt")).read())
print("\n".join(lines))
print("dram bytes/launch", dram)

# ---- the adjoint: launch list of one p2s_backward + p2s_mlp_backward (all four
#      gradients) and one --set full capture of k_adjoint_image (tools/ncu_adjoint_run.sh)
adj_csv = os.path.join(OUT, "adj_launches.csv")
adj_rep = os.path.join(OUT, "prof_adjoint.ncu-rep")
if os.path.exists(adj_csv) and os.path.exists(adj_rep):
    rows = list(csv.reader(open(adj_csv)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(r[ki].split("(")[0], float(r[vi].replace(",", ""))) for r in rows[start + 1:]]
    # the last p2s_backward call of the run (warm-up calls precede it): its kernels in order
    roles = ["(dL/dJ scatter)", "(max |dL/dJ| per plane: U's fp16 range scale)",
             "(MLP + convolutions -> J, dL/dbeta, U = beta dL/dJ)", "(dL/dt)", "(dL/dI)", "(dL/dz)"]
    last = seq[-6:]  # scatter, absmax, fused pass (J, dL/dbeta, U), dL/dt, k_adjoint_image, k_mlp_backward
    raw = subprocess.run(["ncu", "-i", adj_rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    m = {a: (c, b) for a, b, c in zip(rr[0], rr[1], rr[2])}
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__cluster_dim_x", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
    with open(os.path.join(PROF, f"{tag}_ncu_adjoint.txt"), "w") as f:
        f.write("adjoint (p2s_backward + p2s_mlp_backward, all four gradients, cfg3): ncu --metrics "
                "gpu__time_duration.sum --clock-control none (cold-cache, serialised); last call's launches "
                "(tools/adjoint_time.py 1 all4; full list in " + f"{tag}_adjoint_launches.csv):\n")
        for (name, ns), role in zip(last, roles):
            f.write(f"  {ns / 1e3:9.1f} us  {name.removeprefix('void ').split('(')[0].removeprefix('<unnamed>::'):24s} {role}\n")
        f.write("\nncu --set full --clock-control none -k regex:k_adjoint_image -c 1 (dL/dI of one cfg3 frame)\n\n")
        for k in want:
            if k in m:
                f.write(f"{k:80s} {m[k][0]:>16s} {m[k][1]}\n")
    shutil.copy(adj_csv, os.path.join(PROF, f"{tag}_adjoint_launches.csv"))
    print(open(os.path.join(PROF, f"{tag}_ncu_adjoint.txt")).read())

# ---- dL/dz (tools/ncu_dz_run.sh): the resident and the streamed variant, one --set full capture each
dz = [(os.path.join(OUT, "prof_dz_res.ncu-rep"), "resident variant k_mlp_backward<1> (the default on cfg1-4 MLPs)"),
      (os.path.join(OUT, "prof_dz_str.ncu-rep"), "streamed variant k_mlp_backward_s<1> (the default for 33-256-256-100)")]
if all(os.path.exists(f) for f, _ in dz):
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
    with open(os.path.join(PROF, f"{tag}_ncu_mlp_backward.txt"), "w") as f:
        f.write("dL/dz (p2s_mlp_backward): ncu --set full --clock-control none --import-source on, one launch each "
                "(tools/ncu_dz_run.sh; the first on a cfg3 frame, the second the streamed variant forced on the "
                "same frame's inputs after P2S_MB_MODE handling in tools/dz_time.py)\n")
        for rep, title in dz:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rr = list(csv.reader(raw.splitlines()))
            m = {a: (c, b) for a, b, c in zip(rr[0], rr[1], rr[2])}
            f.write(f"\n{title}\n")
            for k in want:
                if k in m:
                    f.write(f"  {k:80s} {m[k][0]:>16s} {m[k][1]}\n")
        if os.path.exists(os.path.join(OUT, "dz_time.log")):
            f.write("\nTiming without ncu (tools/dz_time.py, CUDA events, median of 20): " +
                    open(os.path.join(OUT, "dz_time.log")).read().strip().splitlines()[-1] + "\n")
    print(open(os.path.join(PROF, f"{tag}_ncu_mlp_backward.txt")).read())
