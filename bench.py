#!/usr/bin/env python
"""bench.py — frames/s of the P2S hot path (MLP + Eq. 5 basis convolution + tilt warp) on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on): 512x512 RGB frame,
33 Zernike coefficients per pixel, MLP 33->200->200->K=100, K=100 basis of 33x33 taps, tilt
std 2 px. One step = one p2s_render of one frame per GPU (inputs resident in HBM).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}] [--dry-run]

Prints ONE JSON line (rank 0). N>1: every rank renders its own frames (batch sharding, no
collective on the data path), value = frames of all ranks / max time over
ranks. Under torchrun the world comes from the environment; `--gpus N` without torchrun
re-launches itself under `torch.distributed.run` with N processes (127.0.0.1 rendezvous).
``--impl reference`` times the CPU oracle (oracle/, the stated baseline) on the host cores on
FULL frames of the same workload. ``--dry-run`` exercises the launcher and the rank plumbing
(gloo, no CUDA) and prints the line shape with null measurements.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
N_FUSED = 40  # event-bracketed renders of the dedicated fused-kernel timing loop (roofline)
METRIC = "frames/s and output Mpix/s (512x512 RGB, K=100); tensor-pipe % of peak"
PAPER_CONTEXT = ("Paper: 0.026 s per 256x256 frame (whole simulator, Tesla V100, precision not "
                 "stated; PAPER.md:514/500). Hardie et al. split-step: 24.36 s per frame (PAPER.md:511).")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp["bf16_tflops"], mp.get("bf16_tflops_sustained"), mp["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons sampled every ~2 ms during the run
    (NVML, the library nvidia-smi reads; B200_PROFILING.md's clocks line), with host timestamps;
    `summary(t0, t1)` summarises a window (the main timed region, or every leg of the run).
    Falls back to `nvidia-smi -lms 20` when NVML is unavailable."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, pci_bus_id: str | None = None, period_s: float = 0.002):
        self.idx, self.pci, self.period = gpu_index, pci_bus_id, period_s
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.samples = []  # (host time, sm MHz, max sm MHz, power W, set of reason names)
        self.source = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByPciBusId(self.pci) if self.pci else nv.nvmlDeviceGetHandleByIndex(self.idx)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.time(), float(sm), float(mx), pw,
                                             {n for n, b in bits.items() if rs & b}))
                    except Exception:
                        pass
                    time.sleep(self.period)
            self.nvml = nv
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.source = f"NVML every {self.period * 1e3:.0f} ms"
            return self
        except Exception:
            self.nvml = None
        try:  # fallback: nvidia-smi every 20 ms
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self.source = "nvidia-smi -lms 20"
            deadline = time.time() + 5
            while not self.samples and time.time() < deadline:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.strip().split(",")]
            if len(f) < 10:
                continue
            try:
                self.samples.append((time.time(), float(f[2]), float(f[3]), float(f[4]),
                                     {n for n, v in zip(self.NAMES, f[6:10]) if v.lower().startswith("active")}))
            except ValueError:
                continue

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, pw, mx, reasons = [], [], None, set()
        for ts, c, m, p, rs in list(self.samples):
            if t0 is not None and not (t0 - 0.002 <= ts <= (t1 if t1 is not None else ts) + 0.002):
                continue
            sm.append(c)
            mx = m
            pw.append(p)
            reasons |= rs
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0,
                    "source": self.source}
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(pw) if pw else None,
                "source": self.source}


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_full_frames(spec, frames, threads):
    """Times the oracle (as it stands) on whole frames of `spec`: (seconds per frame list, sample text)."""
    import oracle
    oracle.build()
    times = []
    for f in frames:
        inp = synth.make_inputs(spec, frames=range(f, f + 1))
        t0 = time.perf_counter()
        oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, threads=threads)
        times.append(time.perf_counter() - t0)
    sample = (f"{len(times)} full frame(s) of {spec.name} (all {spec.H}x{spec.W} pixels, {spec.C} channels): "
              f"MLP + Eq.5 conv + warp, fp64, {threads} threads, not extrapolated; host: {lscpu_model()}")
    return times, sample


def maybe_relaunch(args) -> None:
    """`--gpus N` (N > 1) outside torchrun: re-exec this script under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def dry_run(args, rank, world):
    """Launcher/rank plumbing without CUDA: gloo group, per-rank frame blocks, max-over-ranks."""
    dist = pdist.init("gloo") if world > 1 else None
    frames = list(pdist.rank_frames(rank, 1))
    t = pdist.max_over_ranks(1.0 + rank, dist)
    gathered = [None] * world
    if dist:
        dist.all_gather_object(gathered, frames)
    else:
        gathered = [frames]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "frames/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dry_run": True, "rank_frames": gathered, "max_over_ranks_probe": t,
                          "config": {"workload": synth.CONFIGS[CFG_ID].name,
                                     "parallelism": f"batch-sharded x{world}"}}))
    pdist.shutdown(dist)


def reference_arm(args, rank, world):
    """--impl reference: the oracle on full cfg3 frames, one frame per step (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    spec = synth.CONFIGS[CFG_ID]
    threads = oracle.default_threads()
    times, sample = oracle_full_frames(spec, range(args.warmup + args.steps), threads)
    timed = np.array(times[args.warmup:])
    v = float(len(timed) / timed.sum())
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(timed.mean() * 1e3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json configs[2] recipe)",
        "config": {"workload": spec.name, "frames_per_step": 1},
        "mpix_per_s": v * spec.H * spec.W / 1e6,
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "oracle",
                         "sample": f"one full frame per step (frame seed = step index); {sample}"},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


class Timer:
    """CUDA-event timing of calls on the render stream, L2 flushed (256 MiB write) before each
    call outside the events.

    The B200 comes out of even a few milliseconds of idle (a host synchronize, host-side work)
    at a lower effective speed and needs ~3-4 ms of back-to-back work to settle: the first ~15
    cfg3 renders after a pause run 227 -> 175 us (measured, P2S_BENCH_DEBUG). So `pre` untimed
    calls are enqueued right before the timed ones, with no host synchronisation in between."""

    def __init__(self, torch, stream, flush):
        self.torch, self.stream, self.flush = torch, stream, flush

    def warm(self, fn, pre, flush=True):
        for i in range(pre):
            if flush:
                self.flush.fill_(float(i))
            fn()

    def calls(self, fn, n, flush=True, pre=3):
        ev0 = [self.torch.cuda.Event(enable_timing=True) for _ in range(n)]
        ev1 = [self.torch.cuda.Event(enable_timing=True) for _ in range(n)]
        self.torch.cuda.synchronize()
        self.warm(fn, pre, flush)
        for i in range(n):
            if flush:
                self.flush.fill_(float(i))
            ev0[i].record(self.stream)
            fn()
            ev1[i].record(self.stream)
        self.torch.cuda.synchronize()
        return np.array([ev0[i].elapsed_time(ev1[i]) for i in range(n)])

    def fused(self, r, fn, n, pre=16, defer=False):
        """The fused MLP+convolution kernel alone: the library records two events right around
        that launch on its stream (p2s_set_profile_events); an outer pair brackets the whole
        render. Events are created (first record) before the loop, so no lazy creation sits
        between the L2 flush and the launch. Returns (fused ms, evented render ms)."""
        mk = lambda: self.torch.cuda.Event(enable_timing=True)  # noqa: E731
        ev = [[mk() for _ in range(4)] for _ in range(n)]
        for e4 in ev:
            for e in e4:
                e.record(self.stream)
        self.torch.cuda.synchronize()
        self.warm(fn, pre)
        for i in range(n):
            self.flush.fill_(float(i))
            r.set_profile_events(ev[i][1], ev[i][2])
            ev[i][0].record(self.stream)
            fn()
            ev[i][3].record(self.stream)
        r.set_profile_events(None, None)

        def result():
            self.torch.cuda.synchronize()
            return (np.array([e[1].elapsed_time(e[2]) for e in ev]), np.array([e[0].elapsed_time(e[3]) for e in ev]))
        if defer:  # the caller keeps the GPU busy and reads the times later
            return result
        return result()


def executed_macs_per_px(info, C):
    """Padded MACs the tensor cores execute per pixel (dims from p2s_get_info): the MLP's padded
    GEMMs plus C channels x N(=K padded) x 16-tap K-steps of the convolution."""
    return (info["in_pad"] * info["h1_pad"] + info["h1_pad"] * info["h2_pad"] + info["h2_pad"] * info["n_pad"]
            + C * info["n_pad"] * info["conv_steps"] * 16)


def roofline_entry(spec, info, fused_ms, peak, peak_src, traffic=None, frames=1):
    """roofline object of a fused-kernel timing: algorithmic FLOPs / event time."""
    med = float(np.median(fused_ms))
    flops = spec.flops_per_frame() * frames
    achieved = flops / (med / 1e3) / 1e12
    exe = 2.0 * executed_macs_per_px(info, spec.C) * spec.H * spec.W * frames / (med / 1e3) / 1e12
    return {"bound": "tensor", "kernel": "k_fused_p2s", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": f"{peak_src} bf16 dense burst; fp16 kind::f16 runs at the bf16 rate",
            "algorithmic_flops_per_launch": flops, "fused_ms_median": med,
            "fused_ms_mean": float(np.mean(fused_ms)), "fused_ms_min": float(np.min(fused_ms)),
            "fused_ms_max": float(np.max(fused_ms)), "fused_launches_timed": int(len(fused_ms)),
            "tensor_pipe_pct_of_peak_executed": 100.0 * exe / peak,
            "tensor_pipe_note": "executed (padded) tcgen05 MMA FLOPs / fused-kernel time / peak; the ncu "
                                "sm__pipe_tensor_cycles_active of a clock-recorded capture is in ncu"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dry-run", action="store_true", help="launcher + rank plumbing only (gloo, no CUDA)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=3, help="full cfg3 frames the oracle renders for cpu_baseline")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-path leg (profiler launch lists)")
    ap.add_argument("--no-extra", action="store_true", help="skip every extra leg (configs / NEXT rows)")
    for leg in ("configs", "anchor-mode", "batch-mode", "sequence-mode", "adjoint-mode", "color-mode"):
        ap.add_argument(f"--no-{leg}", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200" and not args.dry_run:
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    maybe_relaunch(args)
    rank, world, local_rank = pdist.env_rank_world()
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    extra = not args.no_extra

    import torch
    if torch.cuda.device_count() <= local_rank:
        raise SystemExit(f"rank {rank}: no CUDA device {local_rank} (visible: {torch.cuda.device_count()})")
    dist = None
    if world > 1:
        dist = pdist.init("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2107_11627_b200 import p2s

    spec = synth.CONFIGS[CFG_ID]
    peak, peak_sust, hbm, peak_src = _peaks()
    flops_frame = spec.flops_per_frame()

    # each rank renders its own frame (per-frame seeds = rank): weak scaling, no data-path collective
    inp = synth.make_inputs(spec, frames=pdist.rank_frames(rank, 1))
    r = p2s.Renderer(inp.basis, inp.mlp)
    info = r.info()
    B, C, H, W = inp.image.shape
    r.reserve(B, C, H, W)
    img = torch.from_numpy(inp.image).to(dev)
    z = torch.from_numpy(inp.zernike).to(dev)
    t = torch.from_numpy(inp.tilt).to(dev)
    out = torch.empty_like(img)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    tm = Timer(torch, stream, flush)
    ev_s0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    r.render(img, z, t, out=out)  # first call (allocations, lazy init)
    torch.cuda.synchronize()

    props = torch.cuda.get_device_properties(dev)
    pci = (f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
           if hasattr(props, "pci_bus_id") else None)
    with ClockSampler(torch.cuda.current_device(), pci) as clk:
        t_all0 = time.time()
        # the fused kernel alone (roofline): half of the dedicated loop (after its own pre-warm)
        # before the timed steps, half after them
        # the dedicated loop runs the fused kernel alone (p2s_debug_blur: the same launch writing J
        # to a caller buffer, no warp kernel after it), the library's events right around it
        Jbuf = torch.empty_like(img)
        fused_fn = ((lambda: r.render(img, z, t, out=out)) if os.environ.get("P2S_FUSED_LOOP") == "render"
                    else (lambda: r.debug_blur(img, z, out=Jbuf)))
        fused_pre_res = tm.fused(r, fused_fn, N_FUSED // 2, defer=True)
        # W untimed warm-up steps, enqueued back to back right behind the fused loop's work
        for _ in range(args.warmup):
            flush.fill_(1.0)
            r.render(img, z, t, out=out)
        # ---- the timed steps: one p2s_render per step (MLP + conv kernel, then the warp kernel as
        # its programmatic dependent), L2 flushed before each step outside the events
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        tr0 = time.time()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev_s0[i].record(stream)
            r.render(img, z, t, out=out)
            ev_s1[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        tr1 = time.time()
        step_ms = np.array([ev_s0[i].elapsed_time(ev_s1[i]) for i in range(args.steps)])
        fused_pre, evstep_pre = fused_pre_res()
        tot_ms = pdist.max_over_ranks(float(step_ms.sum()), dist, dev)
        value = pdist.throughput(B, world, args.steps, tot_ms)
        ms_per_step = tot_ms / args.steps

        # ---- the fused kernel alone: the second half of the dedicated loop
        fused_post, evstep_post = tm.fused(r, fused_fn, N_FUSED - N_FUSED // 2)
        fused_ms = np.concatenate([fused_pre, fused_post])
        if os.environ.get("P2S_BENCH_DEBUG"):
            print("fused_pre", np.round(fused_pre * 1e3, 1).tolist(), "\nfused_post", np.round(fused_post * 1e3, 1).tolist(),
                  "\nsteps", np.round(step_ms[:40] * 1e3, 1).tolist(), file=sys.stderr)
        evstep_ms = np.concatenate([evstep_pre, evstep_post])

        # ---- e2e: same metric through p2s_render_host (pinned host buffers, copies inside the step)
        e2e_steps = 0 if args.no_e2e else (args.e2e_steps or max(5, min(args.steps, 20)))
        h_img = torch.from_numpy(inp.image).pin_memory().numpy()
        h_z = torch.from_numpy(inp.zernike).pin_memory().numpy()
        h_t = torch.from_numpy(inp.tilt).pin_memory().numpy()
        h_out = torch.empty(inp.image.shape, dtype=torch.float32).pin_memory().numpy()
        e2e_value = None
        if e2e_steps:
            for _ in range(2):
                r.render_host(h_img, h_z, h_t, h_out)
            if dist:
                dist.barrier()
            e_ms = tm.calls(lambda: r.render_host(h_img, h_z, h_t, h_out), e2e_steps)
            e2e_value = pdist.throughput(B, world, e2e_steps, pdist.max_over_ranks(float(e_ms.sum()), dist, dev))
        h2d = inp.image.nbytes + inp.zernike.nbytes + inp.tilt.nbytes
        d2h = h_out.nbytes

        # ---- the other BASELINE configs at full size (cfg2: the paper's own 256x256 timing shape,
        # PAPER.md:500-514; cfg5: 1024x1024, 65x65 taps, MLP 256 wide)
        configs = None
        if extra and not args.no_configs:
            configs = {}
            for cid in (2, 5):
                cs = synth.CONFIGS[cid]
                ci = synth.make_inputs(cs, frames=pdist.rank_frames(rank, 1))
                cr = p2s.Renderer(ci.basis, ci.mlp)
                cr.reserve(*ci.image.shape)
                cimg, cz, ct = (torch.from_numpy(a).to(dev) for a in (ci.image, ci.zernike, ci.tilt))
                cout = torch.empty_like(cimg)
                fn = (lambda cr=cr, cimg=cimg, cz=cz, ct=ct, cout=cout: cr.render(cimg, cz, ct, out=cout))
                for _ in range(3):
                    fn()
                n = 100 if cid == 2 else 20
                c_ms = tm.calls(fn, n, pre=40 if cid == 2 else 3)
                cf_ms, _ = tm.fused(cr, fn, max(30, n // 2), pre=60 if cid == 2 else 3)
                cv = pdist.throughput(1, world, n, pdist.max_over_ranks(float(c_ms.sum()), dist, dev))
                configs[cs.name] = {
                    "value": cv, "unit": "frames/s", "mpix_per_s": cv * cs.H * cs.W / 1e6,
                    "ms_per_frame": float(c_ms.mean()), "steps": n,
                    "roofline": roofline_entry(cs, cr.info(), cf_ms, peak, peak_src),
                    "whole_render_frac": cs.flops_per_frame() / (c_ms.mean() / 1e3) / 1e12 / peak,
                    "config": {"H": cs.H, "W": cs.W, "C": cs.C, "K": cs.K, "S": cs.S,
                               "mlp": [cs.n_in, cs.h1, cs.h2, cs.K]},
                    "l2": "flushed between calls (256 MiB write)"}
                if cid == 2:
                    configs[cs.name]["context"] = "paper: 0.026 s per 256x256 frame on a V100 (PAPER.md:514)"
                    # a 256x256 frame is 512 tiles for 148 SMs (first-tile latency dominates one frame);
                    # 32 frames per call fill the persistent grid
                    nbb = 32
                    bi = synth.make_inputs(cs, frames=pdist.rank_frames(rank, nbb))
                    bimg2, bz2, bt2 = (torch.from_numpy(a).to(dev) for a in (bi.image, bi.zernike, bi.tilt))
                    bout2 = torch.empty_like(bimg2)
                    cr.reserve(*bi.image.shape)
                    fb = (lambda: cr.render(bimg2, bz2, bt2, out=bout2))  # noqa: E731
                    fb()
                    b_ms = tm.calls(fb, 20, pre=10)
                    bf_ms, _ = tm.fused(cr, fb, 20, pre=10)
                    bv = pdist.throughput(nbb, world, 20, pdist.max_over_ranks(float(b_ms.sum()), dist, dev))
                    configs[cs.name]["batched"] = {
                        "frames_per_call": nbb, "value": bv, "unit": "frames/s", "mpix_per_s": bv * cs.H * cs.W / 1e6,
                        "ms_per_call": float(np.median(b_ms)),
                        "roofline": roofline_entry(cs, cr.info(), bf_ms, peak, peak_src, frames=nbb)}
                    del bimg2, bz2, bt2, bout2
                cr.close()
                del cimg, cz, ct, cout
            torch.cuda.empty_cache()

        # ---- batched launch (the cfg4 shape): 16 frames per p2s_render call,
        # one persistent launch over (frame, tile)
        batch_mode = None
        if extra and not args.no_batch_mode:
            nb = 16
            binp = synth.make_inputs(synth.CONFIGS[4], frames=pdist.rank_frames(rank, nb))
            bimg, bz, bt = (torch.from_numpy(a).to(dev) for a in (binp.image, binp.zernike, binp.tilt))
            bout = torch.empty_like(bimg)
            r.reserve(nb, C, H, W)
            fn = lambda: r.render(bimg, bz, bt, out=bout)  # noqa: E731  16 x 43 MB of inputs: > L2
            for _ in range(2):
                fn()
            n_b = 10
            b_ms = tm.calls(fn, n_b, flush=False)
            fb_ms, _ = tm.fused(r, fn, 10, pre=2)
            rl = roofline_entry(spec, info, fb_ms, peak, peak_src, frames=nb)
            rl["frac_sustained"] = rl["achieved"] / peak_sust if peak_sust else None
            rl["note"] = ("frac against the burst peak (a ~2.6 ms launch is a short kernel); frac_sustained "
                          "against the 4-s back-to-back peak for reference")
            batch_mode = {"frames_per_call": nb, "value": pdist.throughput(nb, world, n_b, pdist.max_over_ranks(
                float(b_ms.sum()), dist, dev)), "unit": "frames/s", "calls": n_b,
                "note": "cfg4: 16 frames (per-frame seeds) per p2s_render; inputs 688 MB > L2",
                "roofline": rl}
            del bimg, bz, bt, bout
            torch.cuda.empty_cache()

        # ---- sequence mode (50 degraded frames per image)
        sequence_mode = None
        if extra and not args.no_sequence_mode:
            F = 50
            sinp = synth.make_inputs(spec, frames=pdist.rank_frames(rank, F))
            simg = torch.from_numpy(np.ascontiguousarray(sinp.image[:1])).to(dev)
            sz, st_ = torch.from_numpy(sinp.zernike).to(dev), torch.from_numpy(sinp.tilt).to(dev)
            sout = torch.empty((F, C, H, W), device=dev, dtype=torch.float32)
            r.reserve(F, C, H, W)
            fn = lambda: r.render_sequence(simg, sz, st_, out=sout)  # noqa: E731  50 x 35 MB: > L2
            for _ in range(2):
                fn()
            s_ms = tm.calls(fn, 5, flush=False, pre=2)
            sequence_mode = {"frames_per_sequence": F, "value": pdist.throughput(F, world, 5, pdist.max_over_ranks(
                float(s_ms.sum()), dist, dev)), "unit": "frames/s", "calls": 5, "api": "p2s_render_sequence",
                "note": "50 frames of one 512x512 RGB image (per-frame Zernike/tilt); the K convolutions "
                        "are computed once per tile and shared by the frames"}
            del simg, sz, st_, sout
            torch.cuda.empty_cache()

        # ---- adjoint
        adjoint_mode = None
        if extra and not args.no_adjoint_mode:
            aimg, az, at = img, z, t
            ag = torch.from_numpy(synth.make_upstream_grad(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
            res = {}
            for key, wb, wt, wi, wz in (("value", True, True, False, False), ("beta_only", True, False, False, False),
                                        ("image_only", False, False, True, False),
                                        ("all", True, True, True, False), ("zernike_only", False, False, False, True),
                                        ("all_with_zernike", True, True, True, True)):
                fn = (lambda wb=wb, wt=wt, wi=wi, wz=wz: r.backward(aimg, az, at, ag, want_beta=wb, want_tilt=wt,
                                                                    want_image=wi, want_zernike=wz))
                for _ in range(3):
                    fn()
                a_ms = tm.calls(fn, 20, pre=8)
                res[key] = pdist.throughput(1, world, 20, pdist.max_over_ranks(float(a_ms.sum()), dist, dev))
            aanc = torch.from_numpy(synth.make_anchors(spec, 16, frames=pdist.rank_frames(rank, 1))).to(dev)
            fn = lambda: r.backward_anchors(aimg, aanc, at, ag)  # noqa: E731
            for _ in range(3):
                fn()
            a_ms = tm.calls(fn, 20, pre=8)
            res["anchor_chain"] = pdist.throughput(1, world, 20, pdist.max_over_ranks(float(a_ms.sum()), dist, dev))
            adjoint_mode = dict(res, unit="frames/s", api="p2s_backward + p2s_mlp_backward",
                                note="value: dL/dbeta [K,H,W] + dL/dt [2,H,W] of one cfg3 frame (L2 flushed per "
                                     "call); beta_only: scatter + conv-only pass; image_only: dL/dI [C,H,W]; all: "
                                     "the three; zernike_only: dL/dz [n_in,H,W]; all_with_zernike: the four; "
                                     "anchor_chain: dL/dA (G = 16) + dL/dt of render_anchors")
            del ag, aanc

        # ---- colour mode
        color_mode = None
        if extra and not args.no_color_mode:
            cz = torch.from_numpy(synth.make_zernike_color(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
            fn = lambda: r.render_color(img, cz, t, out=out)  # noqa: E731
            for _ in range(3):
                fn()
            c_ms = tm.calls(fn, 20, pre=10)
            cg = torch.from_numpy(synth.make_upstream_grad(spec, frames=pdist.rank_frames(rank, 1))).to(dev)
            fa = lambda: r.backward_color(img, cz, t, cg, want_image=True, want_zernike=True)  # noqa: E731
            for _ in range(2):
                fa()
            ca_ms = tm.calls(fa, 10)
            color_mode = {"value": pdist.throughput(1, world, 20, pdist.max_over_ranks(float(c_ms.sum()), dist, dev)),
                          "unit": "frames/s", "calls": 20, "api": "p2s_render_color",
                          "adjoint_value": pdist.throughput(1, world, 10, pdist.max_over_ranks(
                              float(ca_ms.sum()), dist, dev)),
                          "adjoint_api": "p2s_backward_color (all four gradients)",
                          "note": "cfg3 frame, per-channel Zernike fields (z * 540/lambda, lambda = 570/540/450 nm)"}
            del cz, cg

        # ---- anchor-grid mode and the sampler (NEXT-3)
        anchor_mode = None
        if extra and not args.no_anchor_mode:
            G = 16
            anc_h = synth.make_anchors(spec, G, frames=pdist.rank_frames(rank, 1))
            anc = torch.from_numpy(anc_h).to(dev)
            fn = lambda: r.render_anchors(img, anc, t, out=out)  # noqa: E731
            for _ in range(3):
                fn()
            a_ms = tm.calls(fn, 50, pre=20)
            smp = p2s.Sampler(G, spec.n_in, 2.0)
            fs = lambda: (smp.sample(1000 + rank, 0, 1, out=anc), r.render_anchors(img, anc, t, out=out))  # noqa
            for _ in range(2):
                fs()
            sa_ms = tm.calls(fs, 50, pre=20)
            smp.close()
            # NEXT-3 with a dense pre-computed 4096 x 4096 correlation (G = 64, the
            # non-separable exponential stand-in): 50 frames per call on the tensor cores, and the
            # whole simulator per frame (draw + render_anchors at G = 64)
            GD, FD = 64, 50
            dsmp = p2s.Sampler(GD, spec.n_in, spatial_cov=synth.anchor_cov_exp(GD, 6.0))
            danc = torch.empty((FD, spec.n_in, GD, GD), device=dev, dtype=torch.float32)
            fd = lambda: dsmp.sample(7 + rank, 0, FD, out=danc)  # noqa: E731
            for _ in range(2):
                fd()
            d_ms = tm.calls(fd, 10)
            d1 = danc[:1]
            fdr = lambda: (dsmp.sample(7 + rank, 0, 1, out=d1), r.render_anchors(img, d1, t, out=out))  # noqa: E731
            for _ in range(2):
                fdr()
            dr_ms = tm.calls(fdr, 20, pre=20)
            GG2 = GD * GD
            dflops = 2.0 * GG2 * (GG2 + 1) / 2 * FD * spec.n_in  # L's lower triangle x (frame, mode) columns
            dense_sampler = {
                "G": GD, "frames_per_call": FD, "ms_per_call": float(np.median(d_ms)),
                "frames_per_s": pdist.throughput(FD, world, 10, pdist.max_over_ranks(float(d_ms.sum()), dist, dev)),
                "gemm_tflops_algorithmic": dflops / (np.median(d_ms) / 1e3) / 1e12,
                "frac_of_peak": dflops / (np.median(d_ms) / 1e3) / 1e12 / peak,
                "note": "k_draw_y (Philox + mode mixing, fp64) + k_sample_dense (tcgen05, 3 fp16 products per "
                        "K-step: executed MMA = 3x the algorithmic triangle FLOPs)",
                "sample_and_render_fps": pdist.throughput(1, world, 20, pdist.max_over_ranks(float(dr_ms.sum()), dist, dev))}
            dsmp.close()
            del danc, d1
            ae = None
            if e2e_steps:
                h_anc = torch.from_numpy(anc_h).pin_memory().numpy()
                fe = lambda: r.render_anchors_host(h_img, h_anc, h_t, h_out)  # noqa: E731
                for _ in range(2):
                    fe()
                ae_ms = tm.calls(fe, e2e_steps)
                ae = {"value": pdist.throughput(B, world, e2e_steps, pdist.max_over_ranks(float(ae_ms.sum()), dist, dev)),
                      "unit": "frames/s", "h2d_bytes_per_step": int(inp.image.nbytes + anc_h.nbytes + inp.tilt.nbytes),
                      "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                      "api": "p2s_render_anchors_host (pinned host buffers)"}
            anchor_mode = {"G": G, "value": pdist.throughput(B, world, 50, pdist.max_over_ranks(float(a_ms.sum()), dist, dev)),
                           "unit": "frames/s",
                           "sampled_value": pdist.throughput(B, world, 50, pdist.max_over_ranks(float(sa_ms.sum()), dist, dev)),
                           "sampled_note": "NEXT-3: p2s_sample_anchors (separable stand-in covariance, corr_len 2) + "
                                           "p2s_render_anchors per frame",
                           "steps": 50, "api": "p2s_render_anchors", "e2e": ae, "dense_sampler": dense_sampler,
                           "note": "Zernike coefficients on a 16x16 anchor grid (PAPER.md:292-295), bilinear per "
                                   "mode inside the fused kernel; same frame otherwise"}
            del anc
        t_all1 = time.time()

    if dist:
        dist.barrier()
    if rank != 0:
        pdist.shutdown(dist)
        return

    traffic, ncu = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_fused_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                ncu = json.load(f)
            traffic = ncu.get("dram_bytes_per_launch")
        except Exception:
            ncu = None
    roof = roofline_entry(spec, info, fused_ms, peak, peak_src, traffic=traffic)
    roof["fused_le_step"] = bool(roof["fused_ms_median"] <= ms_per_step)
    roof["fused_timing"] = (f"dedicated loop of {N_FUSED} launches of the fused kernel alone (p2s_debug_blur: the same "
                            "kernel, J to a caller buffer, no warp kernel after it), half before and half after "
                            "the timed steps, each behind an L2 flush and a pre-warm; CUDA events recorded by "
                            "the library right around the launch on its stream")
    roof["evented_render_ms_median"] = float(np.median(evstep_ms))
    roof["fused_share_of_evented_render"] = float(np.median(fused_ms) / np.median(evstep_ms))
    roof["whole_render_frac"] = flops_frame * B / (ms_per_step / 1e3) / 1e12 / peak
    if ncu:
        roof["ncu"] = {k: ncu.get(k) for k in ("tensor_pipe_active_pct", "sm_clock_ghz", "gpu_time_us", "source",
                                               "note") if k in ncu}
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16xf16->f32 (tcgen05 kind::f16)",
        "data": "synthetic (seeded; BASELINE.json configs[2] recipe)",
        "config": {"workload": spec.name, "frames_per_step_per_gpu": B, "H": H, "W": W, "C": C,
                   "K": spec.K, "S": spec.S, "mlp": [spec.n_in, spec.h1, spec.h2, spec.K],
                   "l2": "flushed between steps (256 MiB write outside the timed events)",
                   "parallelism": f"batch-sharded x{world}"},
        "mpix_per_s": value * H * W / 1e6,
        "step_ms": {"median": float(np.median(step_ms)), "min": float(step_ms.min()), "max": float(step_ms.max())},
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "api": "p2s_render_host (pinned host buffers)"},
        "gpu_launches": info["kernels_per_render"] * args.steps,
        "configs": configs,
        "anchor_mode": anchor_mode,
        "batch_mode": batch_mode,
        "sequence_mode": sequence_mode,
        "adjoint_mode": adjoint_mode,
        "color_mode": color_mode,
        "clocks": dict(clk.summary(tr0, tr1), all_legs=clk.summary(t_all0, t_all1)),
        "plan": info,
        "context": PAPER_CONTEXT,
    }
    if not args.no_cpu_baseline and world == 1:  # the oracle baseline: rank 0 at N = 1 only
        import oracle
        threads = oracle.default_threads()
        times, sample = oracle_full_frames(spec, range(args.cpu_frames), threads)
        v = len(times) / sum(times)
        line["cpu_baseline"] = {"value": v, "unit": "frames/s", "cores": threads, "kind": "oracle",
                                "sample": sample, "s_per_frame": [round(x, 3) for x in times]}
        # cfg1 and cfg2 (the paper's 256x256 timing shape) also on one thread
        single = {}
        for cid in (1, 2):
            st, _ = oracle_full_frames(synth.CONFIGS[cid], range(1), 1)
            single[synth.CONFIGS[cid].name] = {"s_per_frame": round(st[0], 4), "threads": 1}
        line["cpu_baseline"]["single_thread_full_frames"] = single
    print(json.dumps(line))
    pdist.shutdown(dist)


if __name__ == "__main__":
    main()
