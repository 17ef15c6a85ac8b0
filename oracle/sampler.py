"""Oracle for correlated anchor-grid sampling. TEST INFRASTRUCTURE ONLY
(imported by tests/ and bench.py's reference leg; never by the product package).

PAPER.md:293-295 (Sec. 3.4): "partition the image into a user-defined grid of anchor points ...
This grid corresponds to a correlation matrix ... which can be pre-computed ... sets of Zernike
coefficients are drawn from the correlation matrix". The paper's correlation (Takato 1995 angle
of arrival statistics) needs parameters the paper does not give, so the stand-in
covariance is separable (reading N3):

    Cov[A_j(a, b), A_j'(a', b')] = R[j][j'] * s(a - a') * s(b - b'),
    s(d) = exp(-d^2 / (2 l^2)) (+ 1e-6 on the diagonal),  a, b anchor rows / columns,

and a frame's anchors are A = (L_R (x) L_s (x) L_s) z with z ~ N(0, I), L the Cholesky factors.
z comes from a counter-based generator, so any frame is reproducible on its own:
  Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3"),
  key = (seed lo, seed hi), counter = (frame, anchor g = a G + b, mode j, 0); of its four words
  x0, x1: u1 = (x0 + 0.5) / 2^32, u2 = (x1 + 0.5) / 2^32, z = sqrt(-2 ln u1) cos(2 pi u2)
  (Box-Muller). Everything here is fp64 numpy.
"""
from __future__ import annotations

import numpy as np

_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32_10(counter, key):
    """Philox4x32 with 10 rounds on arrays: counter uint [..., 4], key uint [..., 2] -> uint64
    array [..., 4] of 32-bit words (the S-box-free multiply/xor bijection of Salmon et al.)."""
    c = np.asarray(counter, dtype=np.uint64) & _MASK
    k = np.asarray(key, dtype=np.uint64) & _MASK
    c0, c1, c2, c3 = c[..., 0], c[..., 1], c[..., 2], c[..., 3]
    k0, k1 = np.broadcast_to(k[..., 0], c0.shape), np.broadcast_to(k[..., 1], c0.shape)
    for _ in range(10):
        p0 = np.uint64(_M0) * c0
        p1 = np.uint64(_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(_MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(_MASK)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + np.uint64(_W0)) & np.uint64(_MASK)
        k1 = (k1 + np.uint64(_W1)) & np.uint64(_MASK)
    return np.stack([c0, c1, c2, c3], -1)


def normals(seed: int, frame: int, G: int, n_in: int) -> np.ndarray:
    """z[g][j] ~ N(0,1), g = a G + b, counter (frame, g, j, 0) (Box-Muller on words 0 and 1)."""
    g, j = np.meshgrid(np.arange(G * G), np.arange(n_in), indexing="ij")
    ctr = np.stack([np.full_like(g, frame), g, j, np.zeros_like(g)], -1)
    key = np.array([seed & _MASK, (seed >> 32) & _MASK], dtype=np.uint64)
    x = philox4x32_10(ctr, key).astype(np.float64)
    u1 = (x[..., 0] + 0.5) / 2.0 ** 32
    u2 = (x[..., 1] + 0.5) / 2.0 ** 32
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def spatial_cov(G: int, corr_len: float) -> np.ndarray:
    """s(a - a') over anchor rows (or columns) 0..G-1, in anchor spacings; corr_len 0 -> identity."""
    d = np.arange(G)[:, None] - np.arange(G)[None, :]
    s = np.exp(-d.astype(np.float64) ** 2 / (2.0 * corr_len ** 2)) if corr_len > 0 else (d == 0).astype(np.float64)
    return s + 1e-6 * np.eye(G)


def default_mode_cov(n_in: int) -> np.ndarray:
    """0.25 I (std 0.5 per mode, the configs' Zernike std)."""
    return 0.25 * np.eye(n_in)


def sample(seed: int, frame0: int, F: int, G: int, n_in: int, corr_len: float, mode_cov=None) -> np.ndarray:
    """Anchors [F][n_in][G][G] (fp64): A_f = (L_R (x) L_s (x) L_s) z_f."""
    R = default_mode_cov(n_in) if mode_cov is None else np.asarray(mode_cov, np.float64)
    Ls = np.linalg.cholesky(spatial_cov(G, corr_len))
    LR = np.linalg.cholesky(R)
    out = np.empty((F, n_in, G, G))
    for f in range(F):
        z = normals(seed, frame0 + f, G, n_in).reshape(G, G, n_in)  # [a][b][k]
        t = z @ LR.T                                  # modes:   t[a][b][j] = sum_k L_R[j][k] z[a][b][k]
        t = np.einsum("ac,cbj->abj", Ls, t)           # rows:    sum_c L_s[a][c] t[c][b][j]
        t = np.einsum("bd,adj->abj", Ls, t)           # columns: sum_d L_s[b][d] t[a][d][j]
        out[f] = t.transpose(2, 0, 1)
    return out


def sample_dense(seed: int, frame0: int, F: int, G: int, n_in: int, spatial_cov, mode_cov=None,
                 is_factor: bool = False) -> np.ndarray:
    """Anchors [F][n_in][G][G] (fp64) from a DENSE pre-computed spatial correlation over the G^2
    anchors ("a correlation matrix of size 64^2 x 64^2 = 4096 x 4096 which can be
    pre-computed ... 4096 sets of Zernike coefficients are drawn from the correlation matrix"):

        Cov[A_j(p), A_j'(p')] = R[j][j'] C[p][p'],  p = a G + b (anchor row a, column b)
        A_f = (L_R (x) L) z_f,  L = cholesky(C) [G^2][G^2],  L_R = cholesky(R)

    with the same normals z_f as `sample` (so C = s (x) s reproduces it). spatial_cov [G^2][G^2];
    is_factor=True: spatial_cov already is the lower Cholesky factor L (upper part ignored)."""
    R = default_mode_cov(n_in) if mode_cov is None else np.asarray(mode_cov, np.float64)
    C = np.asarray(spatial_cov, np.float64)
    L = np.tril(C) if is_factor else np.linalg.cholesky(C)
    LR = np.linalg.cholesky(R)
    out = np.empty((F, n_in, G, G))
    for f in range(F):
        z = normals(seed, frame0 + f, G, n_in)   # [p][k]
        y = z @ LR.T                              # modes:  y[p][j] = sum_k L_R[j][k] z[p][k]
        a = L @ y                                 # space:  a[p][j] = sum_q L[p][q] y[q][j]
        out[f] = a.T.reshape(n_in, G, G)
    return out


def mixed_normals(seed: int, frame: int, G: int, n_in: int, mode_cov=None) -> np.ndarray:
    """y [G^2][n_in] = z L_R^T of one frame (the right-hand side sample_dense multiplies by L)."""
    R = default_mode_cov(n_in) if mode_cov is None else np.asarray(mode_cov, np.float64)
    return normals(seed, frame, G, n_in) @ np.linalg.cholesky(R).T

