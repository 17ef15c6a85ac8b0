"""ctypes wrapper of the CPU oracle (oracle/p2s_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg. The product package never imports it.

Every function takes the seeded inputs of ``paper_2107_11627_b200.synth`` (fp32 numpy
arrays) and returns fp64 results of the definitions quoted in p2s_oracle.cpp
(Eq. 5; PAPER.md:280-283 P2S; PAPER.md:172 tilt after blur).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "p2s_oracle.cpp")
_LIB = os.path.join(_HERE, "libp2s_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C++17, -O3 -march=native, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O3", "-march=native", "-ffp-contract=off", "-std=c++17", "-shared", "-fPIC",
                               "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        f = ctypes.POINTER(ctypes.c_float)
        d = ctypes.POINTER(ctypes.c_double)
        i = ctypes.c_int
        common = [f, i, i, i, i, f, i, f, f, i, i, i, i, f, f, f, f, f, f]
        lib.p2s_oracle_beta.argtypes = common + [i, i, d, i]
        lib.p2s_oracle_render.argtypes = common + [i, i, d, d, i]
        lib.p2s_oracle_pixels.argtypes = common + [ctypes.POINTER(ctypes.c_int), i, d, d, i]
        lib.p2s_oracle_warp.argtypes = [d, i, i, i, i, f, d, i]
        lib.p2s_oracle_interp_anchors.argtypes = [f, i, i, i, i, i, d]
        lib.p2s_oracle_adjoint_blur.argtypes = [f, i, i, i, i, f, i, i, d, d, d, d, i]
        for fn in (lib.p2s_oracle_beta, lib.p2s_oracle_render, lib.p2s_oracle_pixels,
                   lib.p2s_oracle_warp, lib.p2s_oracle_interp_anchors, lib.p2s_oracle_adjoint_blur):
            fn.restype = i
        _lib = lib
    return _lib


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class _Args:
    def __init__(self, image, zernike, tilt, basis, mlp):
        self.image = np.ascontiguousarray(image, np.float32)
        self.zernike = np.ascontiguousarray(zernike, np.float32)
        self.tilt = None if tilt is None else np.ascontiguousarray(tilt, np.float32)
        self.basis = np.ascontiguousarray(basis, np.float32)
        self.mlp = {k: np.ascontiguousarray(v, np.float32) for k, v in mlp.items()}
        B, C, H, W = self.image.shape
        K, S, S2 = self.basis.shape
        assert S == S2 and self.zernike.shape[0] == B and self.zernike.shape[2:] == (H, W)
        if self.tilt is not None:
            assert self.tilt.shape == (B, 2, H, W)
        n_in = self.zernike.shape[1]
        h1, h2 = self.mlp["W1"].shape[0], self.mlp["W2"].shape[0]
        assert self.mlp["W1"].shape == (h1, n_in) and self.mlp["W2"].shape == (h2, h1)
        assert self.mlp["W3"].shape == (K, h2)
        self.dims = (B, C, H, W, n_in, K, S, h1, h2)

    def c(self):
        B, C, H, W, n_in, K, S, h1, h2 = self.dims
        t = _fp(self.tilt) if self.tilt is not None else ctypes.POINTER(ctypes.c_float)()
        m = self.mlp
        return [_fp(self.image), B, C, H, W, _fp(self.zernike), n_in, t, _fp(self.basis), K, S,
                h1, h2, _fp(m["W1"]), _fp(m["b1"]), _fp(m["W2"]), _fp(m["b2"]), _fp(m["W3"]),
                _fp(m["b3"])]


def beta(image, zernike, basis, mlp, rows=None, threads=None) -> np.ndarray:
    """Step a1 (P2S MLP): beta [B][K][H][W] fp64."""
    a = _Args(image, zernike, None, basis, mlp)
    B, C, H, W, n_in, K, S, h1, h2 = a.dims
    y0, y1 = rows if rows else (0, H)
    out = np.zeros((B, K, H, W), np.float64)
    rc = _load().p2s_oracle_beta(*a.c(), y0, y1, _dp(out), threads or default_threads())
    assert rc == 0
    return out


def render(image, zernike, tilt, basis, mlp, rows=None, want_blur=False, threads=None):
    """Steps a1-a3: (out, J) fp64 [B][C][H][W]; J (blur before warp) only if want_blur."""
    a = _Args(image, zernike, tilt, basis, mlp)
    B, C, H, W, *_ = a.dims
    y0, y1 = rows if rows else (0, H)
    out = np.zeros((B, C, H, W), np.float64)
    J = np.zeros((B, C, H, W), np.float64) if want_blur else None
    rc = _load().p2s_oracle_render(*a.c(), y0, y1, _dp(J) if J is not None else
                                   ctypes.POINTER(ctypes.c_double)(), _dp(out),
                                   threads or default_threads())
    assert rc == 0
    return out, J


def render_color(image, zernike_c, tilt, basis, mlp, rows=None, want_blur=False, threads=None):
    """Wavelength-dependent colour ("3 PSFs with wavelengths
    450nm, 540nm, and 570nm ... requires 3x computation"): channel c of every frame is rendered as a
    one-channel image with its own Zernike field zernike_c[b][c] -- its own beta, so its own PSF
    field -- and the frame's tilt. zernike_c: [B][C][n_in][H][W]. Returns (out, J) like render."""
    image = np.asarray(image)
    B, C, H, W = image.shape
    out = np.zeros((B, C, H, W), np.float64)
    J = np.zeros((B, C, H, W), np.float64) if want_blur else None
    for c in range(C):
        o, j = render(np.ascontiguousarray(image[:, c:c + 1]), np.ascontiguousarray(zernike_c[:, c]), tilt, basis,
                      mlp, rows=rows, want_blur=want_blur, threads=threads)
        out[:, c] = o[:, 0]
        if want_blur:
            J[:, c] = j[:, 0]
    return out, J


def pixels(image, zernike, tilt, basis, mlp, bxy, want_blur=True, want_out=True, threads=None):
    """Sampled outputs, one by one: (J[n][C], out[n][C]) fp64 at the (b, y, x) triples."""
    a = _Args(image, zernike, tilt, basis, mlp)
    C = a.dims[1]
    bxy = np.ascontiguousarray(bxy, np.int32).reshape(-1, 3)
    n = bxy.shape[0]
    J = np.zeros((n, C), np.float64) if want_blur else None
    out = np.zeros((n, C), np.float64) if want_out else None
    nul = ctypes.POINTER(ctypes.c_double)()
    rc = _load().p2s_oracle_pixels(*a.c(), bxy.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n,
                                   _dp(J) if J is not None else nul,
                                   _dp(out) if out is not None else nul,
                                   threads or default_threads())
    assert rc == 0
    return J, out


def warp(J, tilt, threads=None) -> np.ndarray:
    """Step a3 alone on a given J [B][C][H][W]: fp64."""
    J = np.ascontiguousarray(J, np.float64)
    B, C, H, W = J.shape
    t = None if tilt is None else np.ascontiguousarray(tilt, np.float32)
    out = np.zeros_like(J)
    rc = _load().p2s_oracle_warp(_dp(J), B, C, H, W,
                                 _fp(t) if t is not None else ctypes.POINTER(ctypes.c_float)(),
                                 _dp(out), threads or default_threads())
    assert rc == 0
    return out


def interp_anchors(anchors, H, W) -> np.ndarray:
    """Anchor grid [B][n_in][G][G] -> dense Zernike field [B][n_in][H][W] (fp64), bilinear per
    mode with the corner / half-pixel registration of p2s_oracle.cpp."""
    a = np.ascontiguousarray(anchors, np.float32)
    B, n_in, G, G2 = a.shape
    assert G == G2
    out = np.zeros((B, n_in, H, W), np.float64)
    rc = _load().p2s_oracle_interp_anchors(_fp(a), B, n_in, G, H, W, _dp(out))
    assert rc == 0
    return out


def adjoint_blur(image, basis, beta, gJ, want_beta=True, want_image=True, threads=None):
    """Adjoint of step a2 (Eq. 5 transposed) in the C oracle:
    (dL/dbeta [B][K][H][W] | None, dL/dI [B][C][H][W] | None), fp64, for beta [B][K][H][W] and
    dL/dJ = gJ [B][C][H][W] (see p2s_oracle.cpp)."""
    image = np.ascontiguousarray(image, np.float32)
    basis = np.ascontiguousarray(basis, np.float32)
    beta = np.ascontiguousarray(beta, np.float64)
    gJ = np.ascontiguousarray(gJ, np.float64)
    B, C, H, W = image.shape
    K, S, _ = basis.shape
    assert beta.shape == (B, K, H, W) and gJ.shape == (B, C, H, W)
    gb = np.zeros((B, K, H, W)) if want_beta else None
    gi = np.zeros((B, C, H, W)) if want_image else None
    nul = ctypes.POINTER(ctypes.c_double)()
    rc = _load().p2s_oracle_adjoint_blur(_fp(image), B, C, H, W, _fp(basis), K, S, _dp(beta), _dp(gJ),
                                         _dp(gb) if gb is not None else nul, _dp(gi) if gi is not None else nul,
                                         threads or default_threads())
    assert rc == 0
    return gb, gi

