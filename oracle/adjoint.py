"""Oracle for the adjoint of steps a2-a3. TEST INFRASTRUCTURE ONLY.

The paper presents the simulator as usable "as a differentiable module". For the
forward map of p2s_oracle.cpp written with beta as an input (steps a2-a3, fp64, numpy):

    C_kc(y,x) = sum_{i,j} phi_k[i][j] I_c[cY(y-(i-r))][cX(x-(j-r))]      (true conv, replicate)
    J_c(y,x)  = sum_k beta_k(y,x) C_kc(y,x)                              (Eq. 5, gather)
    out_c(p)  = bilinear(J_c, p - t(p)), clamp-to-edge

and an upstream gradient g = dL/dout, the adjoint quantities are

    dL/dJ_c(q)    = sum_p g_c(p) w_q(p)       (w_q(p): the bilinear weight out_c(p) gives J_c(q))
    dL/dbeta_k(p) = sum_c dL/dJ_c(p) C_kc(p)
    dL/dt_x(p)    = -sum_c g_c(p) d bilinear / d sx, likewise y (0 where the coordinate clamp is
                    active; the derivative of the bilinear weights inside the cell)

`forward_from_beta` and `backward` below are written independently (the backward is not derived
by automatic differentiation); tests/test_oracle_pins.py pins `backward` by central finite
differences of `forward_from_beta` and by the dot-product identity <g, A d> = <A^T g, d>.
"""
from __future__ import annotations

import numpy as np


def _clamp(v, lo, hi):
    return np.minimum(np.maximum(v, lo), hi)


def conv_all(image: np.ndarray, basis: np.ndarray) -> np.ndarray:
    """C [K][C][H][W] (fp64): every basis filter on every channel, true convolution, replicate."""
    C_, H, W = image.shape
    K, S, _ = basis.shape
    r = (S - 1) // 2
    out = np.zeros((K, C_, H, W))
    ys, xs = np.arange(H), np.arange(W)
    for i in range(S):
        for j in range(S):
            yy = _clamp(ys - (i - r), 0, H - 1)
            xx = _clamp(xs - (j - r), 0, W - 1)
            shifted = image[:, yy][:, :, xx].astype(np.float64)  # [C][H][W]
            out += basis[:, i, j].astype(np.float64)[:, None, None, None] * shifted[None]
    return out


def _warp_coords(tilt, H, W):
    y, x = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    sy_raw = y - tilt[1].astype(np.float64)
    sx_raw = x - tilt[0].astype(np.float64)
    sy, sx = _clamp(sy_raw, -1.0, float(H)), _clamp(sx_raw, -1.0, float(W))
    y0, x0 = np.floor(sy), np.floor(sx)
    fy, fx = sy - y0, sx - x0
    y0, x0 = y0.astype(int), x0.astype(int)
    ya, yb = _clamp(y0, 0, H - 1), _clamp(y0 + 1, 0, H - 1)
    xa, xb = _clamp(x0, 0, W - 1), _clamp(x0 + 1, 0, W - 1)
    inside_y = (sy_raw > -1.0) & (sy_raw < H)
    inside_x = (sx_raw > -1.0) & (sx_raw < W)
    return ya, yb, xa, xb, fy, fx, inside_y, inside_x


def forward_from_beta(image, beta, tilt, basis):
    """(out [C][H][W], J [C][H][W], Ck [K][C][H][W]) of one frame, beta [K][H][W] given."""
    Ck = conv_all(image, basis)
    J = np.einsum("khw,kchw->chw", beta.astype(np.float64), Ck)
    C_, H, W = J.shape
    ya, yb, xa, xb, fy, fx, _, _ = _warp_coords(tilt, H, W)
    out = ((1 - fy) * (1 - fx) * J[:, ya, xa] + (1 - fy) * fx * J[:, ya, xb] +
           fy * (1 - fx) * J[:, yb, xa] + fy * fx * J[:, yb, xb])
    return out, J, Ck


def backward(image, beta, tilt, basis, g):
    """(dL/dJ [C][H][W], dL/dbeta [K][H][W], dL/dt [2][H][W]) for upstream g [C][H][W]."""
    _, J, Ck = forward_from_beta(image, beta, tilt, basis)
    C_, H, W = J.shape
    g = g.astype(np.float64)
    ya, yb, xa, xb, fy, fx, in_y, in_x = _warp_coords(tilt, H, W)
    gJ = np.zeros_like(J)
    for (yy, xx, w) in ((ya, xa, (1 - fy) * (1 - fx)), (ya, xb, (1 - fy) * fx),
                        (yb, xa, fy * (1 - fx)), (yb, xb, fy * fx)):
        for c in range(C_):
            np.add.at(gJ[c], (yy, xx), g[c] * w)
    gbeta = np.einsum("chw,kchw->khw", gJ, Ck)
    # d out / d sx = (1-fy)(J[ya][xb] - J[ya][xa]) + fy (J[yb][xb] - J[yb][xa]); sx = x - t_x
    dsx = (1 - fy) * (J[:, ya, xb] - J[:, ya, xa]) + fy * (J[:, yb, xb] - J[:, yb, xa])
    dsy = (1 - fx) * (J[:, yb, xa] - J[:, ya, xa]) + fx * (J[:, yb, xb] - J[:, ya, xb])
    gt = np.zeros((2, H, W))
    gt[0] = -np.where(in_x, (g * dsx).sum(0), 0.0)
    gt[1] = -np.where(in_y, (g * dsy).sum(0), 0.0)
    return gJ, gbeta, gt
