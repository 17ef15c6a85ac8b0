#!/usr/bin/env python
"""bench.py — frames/s of the P2S hot path (MLP + Eq. 5 basis convolution + tilt warp) on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on): 512x512 RGB frame,
33 Zernike coefficients per pixel, MLP 33->200->200->K=100, K=100 basis of 33x33 taps, tilt
std 2 px. One step = one p2s_render of one frame per GPU (inputs resident in HBM).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]

Prints ONE JSON line (rank 0). N>1 runs under torchrun: every rank renders its own frames
(batch sharding, no collective on the data path), value = frames of all ranks / max time.
``--impl reference`` times the CPU oracle (oracle/, the stated baseline) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2107_11627_b200 import dist as pdist  # noqa: E402
from paper_2107_11627_b200 import synth  # noqa: E402

CFG_ID = 3
FUSED_EVERY = 10  # steps per fused-kernel event pair (roofline timing; see the timed loop)
METRIC = "frames/s and output Mpix/s (512x512 RGB, K=100); tensor-pipe % of peak"
PAPER_CONTEXT = ("Paper: 0.026 s per 256x256 frame (whole simulator, Tesla V100, precision not "
                 "stated; PAPER.md:514/500). Hardie et al. split-step: 24.36 s per frame (PAPER.md:511).")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp["bf16_tflops"], mp.get("bf16_tflops_sustained"), mp["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md).

    Sampling starts before the region (waiting for the first sample) and only samples whose
    timestamps fall inside [mark_start, mark_end] are summarised."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 5
            while not self.lines and time.time() < deadline:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if self.t0 is not None and not (self.t0 <= ts <= (self.t1 or ts) + 0.06):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                sm.append(float(f[2]))
                mx = float(f[3])
                pw.append(float(f[4]))
            except ValueError:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


def cpu_reference(spec, inp, budget_s: float, threads: int):
    """Times the oracle (as it stands) on a bounded band of rows of frame 0; frames/s."""
    import oracle
    oracle.build()
    H = spec.H

    def run(rows):
        t0 = time.perf_counter()
        oracle.render(inp.image[:1], inp.zernike[:1], inp.tilt[:1], inp.basis, inp.mlp,
                      rows=(H // 2 - rows // 2, H // 2 - rows // 2 + rows), threads=threads)
        return time.perf_counter() - t0

    probe_rows = 4
    tp = run(probe_rows)
    rows = int(min(H, max(probe_rows, budget_s / max(tp, 1e-6) * probe_rows)))
    t = run(rows) if rows != probe_rows else tp
    fps = (rows / H) / t
    sample = (f"rows [{H // 2 - rows // 2}, {H // 2 - rows // 2 + rows}) of frame 0 ({rows}/{H} rows = "
              f"{rows / H:.3f} frame) of {spec.name}: full MLP + Eq.5 conv (+ the J rows the warp "
              f"reads) + warp, fp64, {threads} threads; {t:.2f} s")
    return fps, t, rows, sample


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-path leg (profiler launch lists)")
    ap.add_argument("--no-anchor-mode", action="store_true", help="skip the anchor-grid (NEXT-1) extra leg")
    ap.add_argument("--no-batch-mode", action="store_true", help="skip the 16-frame batched-launch extra leg")
    ap.add_argument("--no-sequence-mode", action="store_true", help="skip the 50-frame sequence extra leg")
    ap.add_argument("--no-adjoint-mode", action="store_true", help="skip the adjoint (NEXT-4) extra leg")
    ap.add_argument("--no-color-mode", action="store_true", help="skip the per-channel beta (row 5) extra leg")
    args = ap.parse_args()

    rank, world, local_rank = pdist.env_rank_world()
    spec = synth.CONFIGS[CFG_ID]
    peak, peak_sust, hbm, peak_src = _peaks()
    flops_frame = spec.flops_per_frame()

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        inp = synth.make_inputs(spec, frames=range(1))
        threads = oracle.default_threads()
        budget = 8.0
        times, fpss = [], []
        for i in range(args.warmup + args.steps):
            fps, t, rows, sample = cpu_reference(spec, inp, budget, threads)
            if i >= args.warmup:
                times.append(t)
                fpss.append(fps)
        v = float(np.mean(fpss))
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": spec.name, "frames_per_step": 1},
                "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "oracle",
                                 "sample": sample + f"; host: {lscpu_model()}"},
                "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    dist = None
    if world > 1:
        dist = pdist.init("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2107_11627_b200 import p2s

    # each rank renders its own frame (per-frame seeds = rank): weak scaling, no data-path collective
    inp = synth.make_inputs(spec, frames=pdist.rank_frames(rank, 1))
    r = p2s.Renderer(inp.basis, inp.mlp)
    B, C, H, W = inp.image.shape
    r.reserve(B, C, H, W)
    img = torch.from_numpy(inp.image).to(dev)
    z = torch.from_numpy(inp.zernike).to(dev)
    t = torch.from_numpy(inp.tilt).to(dev)
    out = torch.empty_like(img)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    ev_f0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_f1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_s0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    for _ in range(args.warmup):
        flush.fill_(1.0)
        r.render(img, z, t, out=out)
    torch.cuda.synchronize()

    with ClockSampler(torch.cuda.current_device()) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark_start()
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush outside the timed step
            # every FUSED_EVERY-th step brackets the fused kernel with events (roofline); an event
            # between the two kernels stops the warp kernel's programmatic (overlapped) launch,
            # so those steps run ~8 us slower and `value` (all steps) is slightly conservative
            r.set_profile_events(*((ev_f0[i], ev_f1[i]) if i % FUSED_EVERY == 0 else (None, None)))
            ev_s0[i].record(stream)
            r.render(img, z, t, out=out)
            ev_s1[i].record(stream)
        r.set_profile_events(None, None)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall0
        clk.mark_end()
    step_ms = np.array([ev_s0[i].elapsed_time(ev_s1[i]) for i in range(args.steps)])
    inst = [i for i in range(args.steps) if i % FUSED_EVERY == 0]
    fused_ms = np.array([ev_f0[i].elapsed_time(ev_f1[i]) for i in inst])
    clean_step_ms = float(np.mean([step_ms[i] for i in range(args.steps) if i % FUSED_EVERY])) \
        if args.steps > 1 else float(step_ms.mean())
    tot_ms = pdist.max_over_ranks(float(step_ms.sum()), dist, dev)
    value = pdist.throughput(B, world, args.steps, tot_ms)

    # ---- e2e: same metric through p2s_render_host (pinned host buffers, copies inside the step)
    e2e_steps = 0 if args.no_e2e else (args.e2e_steps or max(3, min(args.steps, 10)))
    h_img = torch.from_numpy(inp.image).pin_memory().numpy()
    h_z = torch.from_numpy(inp.zernike).pin_memory().numpy()
    h_t = torch.from_numpy(inp.tilt).pin_memory().numpy()
    h_out = torch.empty(inp.image.shape, dtype=torch.float32).pin_memory().numpy()
    for _ in range(2 if e2e_steps else 0):
        r.render_host(h_img, h_z, h_t, h_out)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(e2e_steps):
        flush.fill_(float(i))
        e0[i].record(stream)
        r.render_host(h_img, h_z, h_t, h_out)
        e1[i].record(stream)
    torch.cuda.synchronize()
    e2e_ms = pdist.max_over_ranks(float(sum(e0[i].elapsed_time(e1[i]) for i in range(e2e_steps))), dist, dev)
    e2e_value = pdist.throughput(B, world, e2e_steps, e2e_ms) if e2e_steps else None
    h2d = inp.image.nbytes + inp.zernike.nbytes + inp.tilt.nbytes
    d2h = h_out.nbytes

    # ---- batched launch (the cfg4 shape): 16 frames per p2s_render call,
    # one persistent launch over (frame, tile) — amortises the ~20 us per-launch fixed cost
    batch_mode = None
    if not args.no_batch_mode:
        nb = 16
        binp = synth.make_inputs(spec, frames=range(rank * nb, (rank + 1) * nb))
        bimg, bz, bt = (torch.from_numpy(a).to(dev) for a in (binp.image, binp.zernike, binp.tilt))
        bout = torch.empty_like(bimg)
        r.reserve(nb, C, H, W)
        for _ in range(2):
            r.render(bimg, bz, bt, out=bout)
        n_b = max(3, min(args.steps // 10, 20))
        b0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_b)]
        b1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_b)]
        torch.cuda.synchronize()
        for i in range(n_b):
            b0[i].record(stream)
            r.render(bimg, bz, bt, out=bout)  # 16 x 43 MB of inputs per call: larger than L2
            b1[i].record(stream)
        torch.cuda.synchronize()
        b_ms = pdist.max_over_ranks(float(sum(b0[i].elapsed_time(b1[i]) for i in range(n_b))), dist, dev)
        # the fused kernel alone over the 16 frames (library events around that launch; separate
        # calls so the timed ones above keep their programmatic warp launch)
        fb0 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        fb1 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for i in range(3):
            r.set_profile_events(fb0[i], fb1[i])
            r.render(bimg, bz, bt, out=bout)
        r.set_profile_events(None, None)
        torch.cuda.synchronize()
        fb_ms = float(np.mean([fb0[i].elapsed_time(fb1[i]) for i in range(3)]))
        fb_tf = flops_frame * nb / (fb_ms * 1e-3) / 1e12
        batch_mode = {"frames_per_call": nb, "value": pdist.throughput(nb, world, n_b, b_ms), "unit": "frames/s",
                      "calls": n_b, "note": "cfg4 shape: 16 frames (cfg3 recipe, per-frame seeds) per p2s_render",
                      "roofline": {"kernel": "k_fused_p2s", "fused_ms_per_call": fb_ms, "achieved": fb_tf,
                                   "unit": "TFLOP/s", "peak_sustained": peak_sust,
                                   "frac_sustained": fb_tf / peak_sust if peak_sust else None,
                                   "frac_burst": fb_tf / peak,
                                   "note": "SURVEY 8(d): long runs (cfg4) against the sustained peak"}}
        del bimg, bz, bt, bout

    # ---- sequence mode (50 degraded frames per image): one
    # image, 50 Zernike fields / tilts; each tile's convolutions serve all 50 frames
    sequence_mode = None
    if not args.no_sequence_mode:
        F = 50
        sinp = synth.make_inputs(spec, frames=range(rank * F, (rank + 1) * F))
        simg = torch.from_numpy(np.ascontiguousarray(sinp.image[:1])).to(dev)
        sz, st_ = torch.from_numpy(sinp.zernike).to(dev), torch.from_numpy(sinp.tilt).to(dev)
        sout = torch.empty((F, C, H, W), device=dev, dtype=torch.float32)
        r.reserve(F, C, H, W)
        for _ in range(2):
            r.render_sequence(simg, sz, st_, out=sout)
        n_s = 5
        q0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_s)]
        q1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_s)]
        torch.cuda.synchronize()
        for i in range(n_s):
            q0[i].record(stream)
            r.render_sequence(simg, sz, st_, out=sout)  # 50 x 35 MB of fields per call: > L2
            q1[i].record(stream)
        torch.cuda.synchronize()
        s_ms = pdist.max_over_ranks(float(sum(q0[i].elapsed_time(q1[i]) for i in range(n_s))), dist, dev)
        sequence_mode = {"frames_per_sequence": F, "value": pdist.throughput(F, world, n_s, s_ms),
                         "unit": "frames/s", "calls": n_s, "api": "p2s_render_sequence",
                         "note": "50 frames of one 512x512 RGB image (cfg3 recipe, per-frame Zernike/tilt); "
                                 "the K convolutions are computed once per tile and shared by the frames"}
        del simg, sz, st_, sout

    # ---- adjoint: dL/dbeta and dL/dt of one cfg3 frame for an upstream
    # gradient (p2s_backward: forward recompute for J, warp-transpose scatter, conv-only fused pass)
    adjoint_mode = None
    if not args.no_adjoint_mode:
        ainp = synth.make_inputs(spec, frames=pdist.rank_frames(rank, 1))
        aimg, az, at = (torch.from_numpy(a).to(dev) for a in (ainp.image, ainp.zernike, ainp.tilt))
        ag = torch.from_numpy(synth.make_upstream_grad(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
        res = {}
        for key, wb, wt, wi, wz in (("value", True, True, False, False), ("beta_only", True, False, False, False),
                                    ("image_only", False, False, True, False),
                                    ("all", True, True, True, False), ("zernike_only", False, False, False, True),
                                    ("all_with_zernike", True, True, True, True)):
            if wz and not r.info()["mlp_backward"]:
                res[key] = None
                continue
            for _ in range(3):
                r.backward(aimg, az, at, ag, want_beta=wb, want_tilt=wt, want_image=wi, want_zernike=wz)
            n_a = max(5, min(args.steps // 4, 50))
            a0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
            a1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
            torch.cuda.synchronize()
            for i in range(n_a):
                flush.fill_(float(i))
                a0[i].record(stream)
                r.backward(aimg, az, at, ag, want_beta=wb, want_tilt=wt, want_image=wi, want_zernike=wz)
                a1[i].record(stream)
            torch.cuda.synchronize()
            a_ms = pdist.max_over_ranks(float(sum(a0[i].elapsed_time(a1[i]) for i in range(n_a))), dist, dev)
            res[key] = pdist.throughput(1, world, n_a, a_ms)
        # the anchor-mode chain (NEXT-1 + NEXT-4): dL/dA (G = 16) + dL/dt through interp ->
        # p2s_backward -> p2s_mlp_backward -> p2s_anchors_backward
        res["anchor_chain"] = None
        if r.info()["mlp_backward"]:
            aanc = torch.from_numpy(synth.make_anchors(spec, 16, frames=pdist.rank_frames(rank, 1))).to(dev)
            for _ in range(3):
                r.backward_anchors(aimg, aanc, at, ag)
            n_a = max(5, min(args.steps // 4, 50))
            a0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
            a1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
            torch.cuda.synchronize()
            for i in range(n_a):
                flush.fill_(float(i))
                a0[i].record(stream)
                r.backward_anchors(aimg, aanc, at, ag)
                a1[i].record(stream)
            torch.cuda.synchronize()
            a_ms = pdist.max_over_ranks(float(sum(a0[i].elapsed_time(a1[i]) for i in range(n_a))), dist, dev)
            res["anchor_chain"] = pdist.throughput(1, world, n_a, a_ms)
            del aanc
        adjoint_mode = {"value": res["value"], "unit": "frames/s", "beta_only": res["beta_only"],
                        "image_only": res["image_only"], "all": res["all"],
                        "zernike_only": res["zernike_only"], "all_with_zernike": res["all_with_zernike"],
                        "anchor_chain": res["anchor_chain"],
                        "api": "p2s_backward + p2s_mlp_backward",
                        "note": "value: dL/dbeta [K,H,W] + dL/dt [2,H,W] of one cfg3 frame (L2 flushed per "
                                "call): dL/dJ scatter, one fused pass (MLP + convolutions -> J, dL/dbeta), "
                                "dL/dt; beta_only: scatter + conv-only pass; image_only: dL/dI [C,H,W] "
                                "(scatter, fused pass -> U = beta dL/dJ, k_adjoint_image); all: the three; zernike_only: "
                                "dL/dz [n_in,H,W] (beta_only's pass, then k_mlp_backward through the MLP); "
                                "all_with_zernike: the four; anchor_chain: dL/dA (G = 16) + dL/dt of render_anchors "
                                "(interp -> p2s_backward -> p2s_mlp_backward -> p2s_anchors_backward)"}
        del aimg, az, at, ag

    # ---- colour mode: per-channel Zernike fields (the
    # frame's field at 570/540/450 nm) -> per-channel beta; one fused launch per frame
    color_mode = None
    if not args.no_color_mode:
        cinp = synth.make_inputs(spec, frames=pdist.rank_frames(rank, 1))
        cimg, ct = (torch.from_numpy(a).to(dev) for a in (cinp.image, cinp.tilt))
        cz = torch.from_numpy(synth.make_zernike_color(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
        cout = torch.empty_like(cimg)
        for _ in range(3):
            r.render_color(cimg, cz, ct, out=cout)
        n_c = max(5, min(args.steps // 4, 50))
        c0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_c)]
        c1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_c)]
        torch.cuda.synchronize()
        for i in range(n_c):
            flush.fill_(float(i))
            c0[i].record(stream)
            r.render_color(cimg, cz, ct, out=cout)
            c1[i].record(stream)
        torch.cuda.synchronize()
        c_ms = pdist.max_over_ranks(float(sum(c0[i].elapsed_time(c1[i]) for i in range(n_c))), dist, dev)
        # its adjoint (p2s_backward_color): dL/dbeta_c, dL/dt, dL/dI and dL/dz_c of the same frame
        cg = torch.from_numpy(synth.make_upstream_grad(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
        adj_v = None
        if r.info()["mlp_backward"]:
            for _ in range(2):
                r.backward_color(cimg, cz, ct, cg, want_image=True, want_zernike=True)
            n_ca = max(3, min(args.steps // 20, 20))
            c0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_ca)]
            c1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_ca)]
            torch.cuda.synchronize()
            for i in range(n_ca):
                flush.fill_(float(i))
                c0[i].record(stream)
                r.backward_color(cimg, cz, ct, cg, want_image=True, want_zernike=True)
                c1[i].record(stream)
            torch.cuda.synchronize()
            ca_ms = pdist.max_over_ranks(float(sum(c0[i].elapsed_time(c1[i]) for i in range(n_ca))), dist, dev)
            adj_v = pdist.throughput(1, world, n_ca, ca_ms)
        color_mode = {"value": pdist.throughput(1, world, n_c, c_ms), "unit": "frames/s", "calls": n_c,
                      "api": "p2s_render_color",
                      "adjoint_value": adj_v, "adjoint_api": "p2s_backward_color (all four gradients)",
                      "note": "cfg3 frame, per-channel Zernike fields (z * 540/lambda, lambda = 570/540/450 nm) "
                              "-> per-channel beta; the convolutions once per tile, 3 MLP + J passes"}
        del cimg, ct, cz, cout, cg

    # ---- anchor-grid mode: the same frame with its Zernike coefficients
    # given on a 16x16 anchor grid and interpolated inside the fused kernel (not the headline
    # workload, which BASELINE.json defines on a dense field); same timing protocol
    anchor_mode = None
    if not args.no_anchor_mode:
        G = 16
        anc_h = synth.make_anchors(spec, G, frames=pdist.rank_frames(rank, 1))
        anc = torch.from_numpy(anc_h).to(dev)
        for _ in range(3):
            r.render_anchors(img, anc, t, out=out)
        n_a = max(10, min(args.steps, 100))
        a0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
        a1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_a)]
        torch.cuda.synchronize()
        for i in range(n_a):
            flush.fill_(float(i))
            a0[i].record(stream)
            r.render_anchors(img, anc, t, out=out)
            a1[i].record(stream)
        torch.cuda.synchronize()
        a_ms = pdist.max_over_ranks(float(sum(a0[i].elapsed_time(a1[i]) for i in range(n_a))), dist, dev)
        # the whole simulator from a seed (NEXT-3 + NEXT-1): correlated anchors, then the frame
        smp = p2s.Sampler(G, spec.n_in, 2.0)
        for _ in range(2):
            r.render_anchors(img, smp.sample(1000 + rank, 0, 1, out=anc), t, out=out)
        torch.cuda.synchronize()
        for i in range(n_a):
            flush.fill_(float(i))
            a0[i].record(stream)
            smp.sample(1000 + rank, i, 1, out=anc)
            r.render_anchors(img, anc, t, out=out)
            a1[i].record(stream)
        torch.cuda.synchronize()
        sa_ms = pdist.max_over_ranks(float(sum(a0[i].elapsed_time(a1[i]) for i in range(n_a))), dist, dev)
        smp.close()
        h_anc = torch.from_numpy(anc_h).pin_memory().numpy()
        ae = None
        if e2e_steps:
            for _ in range(2):
                r.render_anchors_host(h_img, h_anc, h_t, h_out)
            torch.cuda.synchronize()
            for i in range(e2e_steps):
                flush.fill_(float(i))
                e0[i].record(stream)
                r.render_anchors_host(h_img, h_anc, h_t, h_out)
                e1[i].record(stream)
            torch.cuda.synchronize()
            ae_ms = pdist.max_over_ranks(float(sum(e0[i].elapsed_time(e1[i]) for i in range(e2e_steps))), dist, dev)
            ae = {"value": pdist.throughput(B, world, e2e_steps, ae_ms), "unit": "frames/s",
                  "h2d_bytes_per_step": int(inp.image.nbytes + anc_h.nbytes + inp.tilt.nbytes),
                  "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                  "api": "p2s_render_anchors_host (pinned host buffers)"}
        anchor_mode = {"G": G, "value": pdist.throughput(B, world, n_a, a_ms), "unit": "frames/s",
                       "sampled_value": pdist.throughput(B, world, n_a, sa_ms),
                       "sampled_note": "NEXT-3: p2s_sample_anchors (correlated anchors from a seed, stand-in "
                                       "covariance, corr_len 2) + p2s_render_anchors per frame",
                       "steps": n_a, "api": "p2s_render_anchors", "e2e": ae,
                       "note": "SURVEY NEXT-1: Zernike coefficients on a 16x16 anchor grid (PAPER.md:285-288), "
                               "bilinear per mode inside the fused kernel; same frame otherwise"}

    if dist:
        dist.barrier()
    if rank != 0:
        pdist.shutdown(dist)
        return

    fused_mean = float(fused_ms.mean())
    achieved = flops_frame * B / (fused_mean / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_fused_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    info = r.info()
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16xf16->f32 (tcgen05 kind::f16)",
        "data": "synthetic (seeded; BASELINE.json configs[2] recipe)",
        "config": {"workload": spec.name, "frames_per_step_per_gpu": B, "H": H, "W": W, "C": C,
                   "K": spec.K, "S": spec.S, "mlp": [spec.n_in, spec.h1, spec.h2, spec.K],
                   "l2": "flushed between steps (256 MiB write outside the timed events)",
                   "parallelism": f"batch-sharded x{world}"},
        "mpix_per_s": value * H * W / 1e6,
        "roofline": {"bound": "tensor", "kernel": "k_fused_p2s", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{peak_src} bf16 dense (burst); fp16 kind::f16 runs at the same rate",
                     "algorithmic_flops_per_launch": flops_frame * B, "fused_ms_mean": fused_mean,
                     "fused_ms_min": float(fused_ms.min()),
                     "fused_timed_steps": f"every {FUSED_EVERY}th timed step ({len(fused_ms)} of {args.steps})",
                     "clean_step_ms": clean_step_ms,
                     "whole_render_frac": flops_frame * B / (tot_ms / args.steps / 1e3) / 1e12 / peak},
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "api": "p2s_render_host (pinned host buffers)"},
        "gpu_launches": info["kernels_per_render"] * args.steps,
        "anchor_mode": anchor_mode,
        "batch_mode": batch_mode,
        "sequence_mode": sequence_mode,
        "adjoint_mode": adjoint_mode,
        "color_mode": color_mode,
        "clocks": clk.summary(),
        "wall_s": t_wall,
        "plan": info,
        "context": PAPER_CONTEXT,
    }
    if not args.no_cpu_baseline and world == 1:  # the oracle baseline: rank 0 at N = 1 only
        import oracle
        threads = oracle.default_threads()
        fps, tcpu, rows, sample = cpu_reference(spec, inp, args.cpu_budget, threads)
        line["cpu_baseline"] = {"value": fps, "unit": "frames/s", "cores": threads, "kind": "oracle",
                                "sample": sample + f"; host: {lscpu_model()}"}
    print(json.dumps(line))
    pdist.shutdown(dist)


if __name__ == "__main__":
    main()
