"""Seeded synthetic inputs for the P2S hot path (shared by tests, bench and smoke).

This module only *draws* inputs. It holds none of the method's arithmetic (no MLP
evaluation, no convolution, no warp): both the CUDA path and the CPU oracle consume
what it returns, so it is the one piece of code the two may share (task rule ③).

Recipe (DESIGN.md §"Input recipe"; SURVEY.md §8(d) "Synthetic inputs"):

* generator: ``numpy.random.default_rng(SeedSequence([cfg_id, frame, stream]))`` with
  stream ids 0 = image, 1 = Zernike field, 2 = tilt, 3 = basis, 4 = MLP, 5 = rectangles.
  Basis and MLP use frame 0 and are shared by every frame of a batch.
* image: U[0,1) per channel; configs 3-5 paint 8 axis-aligned constant rectangles
  (stand-in for natural-image edges of the paper's Places training images, P:474 — that
  dataset is not available and is not reconstructed).
* Zernike field: ``n_in`` independent N(0,1) HxW fields, smoothed with a periodic
  Gaussian (FFT, sigma px), mean removed, scaled to the exact std. Stand-in for the
  anchor-interpolated correlated Zernike fields of P:293 (Noll/Takato covariances and
  the supplementary turbulence parameters are absent).
* tilt: 2 fields built the same way (ch0 = x / columns, ch1 = y / rows, in pixels).
* basis: G ~ N(0,1)^{S^2 x K} (fp64) -> reduced QR -> columns sign-fixed by diag(R) ->
  phi_k = Q[:, k] reshaped SxS row-major. Stand-in for the PCA basis of P:254.
* MLP: PyTorch-default ``nn.Linear`` init, W, b ~ U(+-1/sqrt(fan_in));
  ``init="he"`` gives the He-normal stress variant (W ~ N(0, 2/fan_in), b = 0).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

STREAM_IMAGE, STREAM_ZERNIKE, STREAM_TILT, STREAM_BASIS, STREAM_MLP, STREAM_RECT, STREAM_ANCHORS, STREAM_GRAD, \
    STREAM_TILE = range(9)


@dataclass(frozen=True)
class Spec:
    """Shape/statistics of one workload (BASELINE.json ``configs`` entries)."""
    name: str
    cfg_id: int
    B: int
    C: int
    H: int
    W: int
    K: int          # number of basis PSFs (the paper's M)
    S: int          # odd tap size of each basis PSF
    n_in: int = 33  # high-order Zernike inputs Z4..Z36
    h1: int = 200
    h2: int = 200
    z_sigma: float = 8.0
    z_std: float = 0.5
    t_sigma: float = 16.0
    t_std: float = 0.0   # 0 => zero tilt field
    rects: int = 0
    init: str = "torch"  # "torch" (default nn.Linear) or "he"

    @property
    def pixels(self) -> int:
        return self.H * self.W

    def mlp_macs_per_px(self) -> int:
        return self.n_in * self.h1 + self.h1 * self.h2 + self.h2 * self.K

    def conv_macs_per_px(self) -> int:
        return self.C * self.K * self.S * self.S

    def flops_per_frame(self) -> float:
        """Algorithmic FLOPs of steps a1+a2 (MLP + basis conv), 2 per MAC."""
        return 2.0 * self.pixels * (self.mlp_macs_per_px() + self.conv_macs_per_px())


# BASELINE.json configs[0..4] (cfg1..cfg5)
CONFIGS = {
    1: Spec("cfg1_64_gray_K16_S15", 1, B=1, C=1, H=64, W=64, K=16, S=15, h1=64, h2=64,
            z_sigma=4, z_std=0.5, t_sigma=16, t_std=0.0, rects=0),
    2: Spec("cfg2_256_gray_K100_S33", 2, B=1, C=1, H=256, W=256, K=100, S=33,
            z_sigma=8, z_std=0.5, t_sigma=16, t_std=1.5, rects=0),
    3: Spec("cfg3_512_rgb_K100_S33", 3, B=1, C=3, H=512, W=512, K=100, S=33,
            z_sigma=16, z_std=0.5, t_sigma=32, t_std=2.0, rects=8),
    4: Spec("cfg4_16x512_rgb_K100_S33", 4, B=16, C=3, H=512, W=512, K=100, S=33,
            z_sigma=16, z_std=0.5, t_sigma=32, t_std=2.0, rects=8),
    5: Spec("cfg5_1024_rgb_K100_S65", 5, B=1, C=3, H=1024, W=1024, K=100, S=65, h1=256, h2=256,
            z_sigma=32, z_std=0.7, t_sigma=64, t_std=4.0, rects=8),
}


def custom(name: str, cfg_id: int, **kw) -> Spec:
    """A test workload (ragged sizes etc.) drawn with the same recipe."""
    base = dict(B=1, C=1, H=32, W=32, K=8, S=7, h1=32, h2=32, z_sigma=4.0, z_std=0.5,
                t_sigma=8.0, t_std=1.0, rects=0)
    base.update(kw)
    return Spec(name, cfg_id, **base)


def _rng(cfg_id: int, frame: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(cfg_id), int(frame), int(stream)]))


def smooth_field(rng: np.random.Generator, n: int, H: int, W: int, sigma: float, std: float) -> np.ndarray:
    """n periodic-Gaussian-smoothed N(0,1) fields, zero-mean, exact std. fp32 [n][H][W]."""
    out = np.empty((n, H, W), np.float32)
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.rfftfreq(W)[None, :]
    g = np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * (fy ** 2 + fx ** 2))
    for i in range(n):
        f = rng.standard_normal((H, W))
        if sigma > 0:
            f = np.fft.irfft2(np.fft.rfft2(f) * g, s=(H, W))
        f = f - f.mean()
        sd = f.std()
        f = f * (std / sd) if sd > 0 else f
        out[i] = f.astype(np.float32)
    return out


def make_image(spec: Spec, frame: int) -> np.ndarray:
    rng = _rng(spec.cfg_id, frame, STREAM_IMAGE)
    img = rng.random((spec.C, spec.H, spec.W), dtype=np.float64)
    if spec.rects:
        rr = _rng(spec.cfg_id, frame, STREAM_RECT)
        H, W = spec.H, spec.W
        for _ in range(spec.rects):
            y0 = int(rr.integers(0, H))
            x0 = int(rr.integers(0, W))
            hh = int(rr.integers(max(1, H // 16), max(2, H // 4) + 1))
            ww = int(rr.integers(max(1, W // 16), max(2, W // 4) + 1))
            val = rr.random(spec.C)
            img[:, y0:y0 + hh, x0:x0 + ww] = val[:, None, None]
    return img.astype(np.float32)


def make_zernike(spec: Spec, frame: int) -> np.ndarray:
    return smooth_field(_rng(spec.cfg_id, frame, STREAM_ZERNIKE), spec.n_in, spec.H, spec.W,
                        spec.z_sigma, spec.z_std)


def make_anchors(spec: Spec, G: int, frames: Optional[range] = None) -> np.ndarray:
    """Anchor-grid Zernike coefficients [B][n_in][G][G] fp32:
    per mode an N(0,1) G x G field, periodic-Gaussian smoothed over ~1 anchor spacing and scaled
    to the config's Zernike std — a stand-in for the spatially correlated draws of P:293 (the
    Takato covariance needs the missing supplementary parameters)."""
    frames = range(spec.B) if frames is None else frames
    return np.stack([smooth_field(_rng(spec.cfg_id, f, STREAM_ANCHORS), spec.n_in, G, G, 1.0, spec.z_std)
                     for f in frames])


def anchor_cov_exp(G: int, corr_len: float, jitter: float = 1e-6) -> np.ndarray:
    """A dense, NON-separable spatial correlation over the G x G anchor grid (fp64 [G^2][G^2],
    p = a G + b): exp(-|p - p'| / corr_len) of the Euclidean anchor distance (in anchor
    spacings) + jitter I. Stand-in for the pre-computed Takato/Chimitt correlation matrix of
    PAPER.md:293-295, whose turbulence parameters the paper does not give (reading N6).
    The exponential (Matern nu = 1/2) kernel is positive definite in 2-D; it is not a Kronecker
    product, so only the dense sampler can draw from it."""
    a, b = np.divmod(np.arange(G * G), G)
    d = np.hypot(a[:, None] - a[None, :], b[:, None] - b[None, :]).astype(np.float64)
    c = np.exp(-d / corr_len) if corr_len > 0 else (d == 0).astype(np.float64)
    return c + jitter * np.eye(G * G)


def anchor_cov_separable(G: int, corr_len: float) -> np.ndarray:
    """The separable stand-in s (x) s of p2s_sampler_init written as a dense [G^2][G^2] matrix
    (s(d) = exp(-d^2 / (2 l^2)) + 1e-6 [d = 0], reading N3)."""
    d = np.arange(G)[:, None] - np.arange(G)[None, :]
    s = np.exp(-d.astype(np.float64) ** 2 / (2.0 * corr_len ** 2)) if corr_len > 0 else (d == 0).astype(np.float64)
    s = s + 1e-6 * np.eye(G)
    return np.kron(s, s)


WAVELENGTHS_NM = (570.0, 540.0, 450.0)  # R, G, B as in PAPER.md:318 ("450nm, 540nm, and 570nm")


def make_zernike_color(spec: Spec, frames: Optional[range] = None, ref_nm: float = 540.0) -> np.ndarray:
    """Per-channel Zernike fields [B][C][n_in][H][W] fp32 for the colour mode: the
    frame's field (make_zernike, defined at ref_nm) seen at each channel's wavelength -- a phase
    aberration in radians scales as 1/lambda, so z_c = z * ref_nm / lambda_c (C = 3: R, G, B at
    570, 540, 450 nm; other C: wavelengths spread evenly over 450..570 nm)."""
    frames = range(spec.B) if frames is None else frames
    lam = WAVELENGTHS_NM if spec.C == 3 else tuple(np.linspace(570.0, 450.0, spec.C))
    return np.stack([np.stack([make_zernike(spec, f) * np.float32(ref_nm / l) for l in lam])
                     for f in frames]).astype(np.float32)


def make_upstream_grad(spec: Spec, frames: Optional[range] = None) -> np.ndarray:
    """dL/dout [B][C][H][W] fp32 for the adjoint: i.i.d. U(-1, 1), the gradient of
    a loss on the rendered frames (no structure assumed)."""
    frames = range(spec.B) if frames is None else frames
    return np.stack([_rng(spec.cfg_id, f, STREAM_GRAD).uniform(-1.0, 1.0, (spec.C, spec.H, spec.W))
                     for f in frames]).astype(np.float32)


def make_tilt(spec: Spec, frame: int) -> np.ndarray:
    if spec.t_std == 0:
        return np.zeros((2, spec.H, spec.W), np.float32)
    return smooth_field(_rng(spec.cfg_id, frame, STREAM_TILT), 2, spec.H, spec.W,
                        spec.t_sigma, spec.t_std)


def make_basis(spec: Spec) -> np.ndarray:
    """[K][S][S] fp32, QR-orthonormal columns (needs S*S >= K)."""
    rng = _rng(spec.cfg_id, 0, STREAM_BASIS)
    T = spec.S * spec.S
    G = rng.standard_normal((T, spec.K))
    Q, R = np.linalg.qr(G, mode="reduced")
    Q = Q * np.sign(np.diag(R))[None, :]
    return np.ascontiguousarray(Q.T.reshape(spec.K, spec.S, spec.S)).astype(np.float32)


def make_mlp(spec: Spec) -> dict:
    """nn.Linear layout: W[out][in], b[out]; fp32."""
    rng = _rng(spec.cfg_id, 0, STREAM_MLP)
    dims = [(spec.h1, spec.n_in), (spec.h2, spec.h1), (spec.K, spec.h2)]
    out = {}
    for li, (o, i) in enumerate(dims, start=1):
        if spec.init == "he":
            w = rng.standard_normal((o, i)) * np.sqrt(2.0 / i)
            b = np.zeros(o)
        else:
            bound = 1.0 / np.sqrt(i)
            w = rng.uniform(-bound, bound, (o, i))
            b = rng.uniform(-bound, bound, o)
        out[f"W{li}"] = np.ascontiguousarray(w, dtype=np.float32)
        out[f"b{li}"] = np.ascontiguousarray(b, dtype=np.float32)
    return out


@dataclass
class Inputs:
    spec: Spec
    image: np.ndarray    # [B][C][H][W] fp32
    zernike: np.ndarray  # [B][n_in][H][W] fp32
    tilt: np.ndarray     # [B][2][H][W] fp32 (px; ch0 = x, ch1 = y)
    basis: np.ndarray    # [K][S][S] fp32
    mlp: dict = field(default_factory=dict)


def make_inputs(spec: Spec, frames: Optional[range] = None) -> Inputs:
    frames = range(spec.B) if frames is None else frames
    img = np.stack([make_image(spec, f) for f in frames])
    z = np.stack([make_zernike(spec, f) for f in frames])
    t = np.stack([make_tilt(spec, f) for f in frames])
    return Inputs(replace(spec, B=len(frames)), img, z, t, make_basis(spec), make_mlp(spec))


# ---- huge frames (maximum-size tests): a base block tiled ry x rx times, every replica scaled by its
# own seeded factors so that no two tiles hold the same values. The full arrays (several GB) are
# only ever built on the device, by indexing alone (the test's `repeat` + two multiplies in this
# order); the host takes crops of the same definition: big[..., y, x] =
# (base[..., y % bh, x % bw] * sy[y // bh]) * sx[x // bw], all in fp32.
def tile_scales(spec: Spec, n: int, axis: int) -> np.ndarray:
    """n per-tile scale factors U[0.75, 1.25) (fp32) for tile rows (axis 0) or columns (axis 1)."""
    return _rng(spec.cfg_id, axis, STREAM_TILE).uniform(0.75, 1.25, n).astype(np.float32)


def tiled_crop(base: np.ndarray, sy: np.ndarray, sx: np.ndarray, y0: int, y1: int, x0: int, x1: int) -> np.ndarray:
    """Rows [y0, y1) x columns [x0, x1) of the tiled array of `base` [..., bh, bw] (fp32)."""
    bh, bw = base.shape[-2:]
    ys, xs = np.arange(y0, y1), np.arange(x0, x1)
    blk = np.asarray(base, np.float32)[..., (ys % bh)[:, None], (xs % bw)[None, :]]
    return (blk * sy[ys // bh][:, None]) * sx[xs // bw][None, :]
