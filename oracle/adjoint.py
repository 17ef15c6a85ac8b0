"""Oracle for the adjoint of steps a2-a3. TEST INFRASTRUCTURE ONLY.

The paper presents the simulator as usable "as a differentiable module". For the
forward map of p2s_oracle.cpp written with beta as an input (steps a2-a3, fp64, numpy):

    C_kc(y,x) = sum_{i,j} phi_k[i][j] I_c[cY(y-(i-r))][cX(x-(j-r))]      (true conv, replicate)
    J_c(y,x)  = sum_k beta_k(y,x) C_kc(y,x)                              (Eq. 5, gather)
    out_c(p)  = bilinear(J_c, p - t(p)), clamp-to-edge

and an upstream gradient g = dL/dout, the adjoint quantities are

    dL/dJ_c(q)    = sum_p g_c(p) w_q(p)       (w_q(p): the bilinear weight out_c(p) gives J_c(q))
    dL/dbeta_k(p) = sum_c dL/dJ_c(p) C_kc(p)
    dL/dI_c(q)    = sum_{p,k,i,j: cY(p_y-(i-r)) = q_y, cX(p_x-(j-r)) = q_x} phi_k[i][j] beta_k(p) dL/dJ_c(p)
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


def _warp_coords(tilt, H, W, coord_dtype=np.float64):
    """Source coordinates s = p - t(p) and their bilinear cell. coord_dtype is the precision s is
    formed in: the cell (an integer) is decided there, and d out/d s jumps across cell edges, so
    the GPU parity tests pass np.float32 -- the kernel's precision (reading N4). The
    weights and everything after them stay fp64."""
    y, x = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    sy_raw = (y.astype(coord_dtype) - tilt[1].astype(coord_dtype)).astype(np.float64)
    sx_raw = (x.astype(coord_dtype) - tilt[0].astype(coord_dtype)).astype(np.float64)
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


def conv_at(image, basis, yx):
    """C_kc at the listed pixels only: [n][K][C] (fp64), the sum of conv_all's definition."""
    C_, H, W = image.shape
    K, S, _ = basis.shape
    r = (S - 1) // 2
    out = np.zeros((len(yx), K, C_))
    for n, (y, x) in enumerate(yx):
        yy = _clamp(y - (np.arange(S) - r), 0, H - 1)
        xx = _clamp(x - (np.arange(S) - r), 0, W - 1)
        patch = image[:, yy][:, :, xx].astype(np.float64)  # [C][i][j] = I_c[cY(y-(i-r))][cX(x-(j-r))]
        out[n] = np.einsum("kij,cij->kc", basis.astype(np.float64), patch)
    return out


def grad_J(tilt, g, coord_dtype=np.float64):
    """dL/dJ [C][H][W]: g scattered through the warp's bilinear weights (the transpose of step a3)."""
    C_, H, W = g.shape
    g = g.astype(np.float64)
    ya, yb, xa, xb, fy, fx, _, _ = _warp_coords(tilt, H, W, coord_dtype)
    gJ = np.zeros((C_, H, W))
    for (yy, xx, w) in ((ya, xa, (1 - fy) * (1 - fx)), (ya, xb, (1 - fy) * fx),
                        (yb, xa, fy * (1 - fx)), (yb, xb, fy * fx)):
        for c in range(C_):
            np.add.at(gJ[c], (yy, xx), g[c] * w)
    return gJ


def grad_image(beta, basis, gJ):
    """dL/dI [C][H][W]: the transpose of step a2 (the beta-weighted convolution, scatter order):
    every term phi_k[i][j] I[cY(y-(i-r))][cX(x-(j-r))] of J_c(y,x) sends
    phi_k[i][j] beta_k(y,x) dL/dJ_c(y,x) back to the (clamped) pixel it read."""
    C_, H, W = gJ.shape
    K, S, _ = basis.shape
    r = (S - 1) // 2
    out = np.zeros((C_, H, W))
    ys, xs = np.arange(H), np.arange(W)
    for i in range(S):
        yy = _clamp(ys - (i - r), 0, H - 1)
        for j in range(S):
            xx = _clamp(xs - (j - r), 0, W - 1)
            v = np.einsum("k,khw->hw", basis[:, i, j].astype(np.float64), beta.astype(np.float64))
            for c in range(C_):
                np.add.at(out[c], (yy[:, None], xx[None, :]), v * gJ[c])
    return out


def _preimage(q, d, n):
    """{p in [0, n) : clamp(p - d, 0, n - 1) == q}: the pixels whose tap at offset d read q."""
    if q == 0:
        return np.arange(0, max(0, min(n - 1, d) + 1))
    if q == n - 1:
        return np.arange(min(n, max(0, n - 1 + d)), n)
    p = q + d
    return np.array([p]) if 0 <= p < n else np.arange(0)


def grad_image_at(beta, basis, gJ, yx):
    """grad_image at the listed pixels only: [n][C] (fp64), by the same definition (each tap's
    preimage under the clamp is a rectangle of output pixels)."""
    C_, H, W = gJ.shape
    K, S, _ = basis.shape
    r = (S - 1) // 2
    out = np.zeros((len(yx), C_))
    for n, (y, x) in enumerate(yx):
        for i in range(S):
            rows = _preimage(y, i - r, H)
            if rows.size == 0:
                continue
            for j in range(S):
                cols = _preimage(x, j - r, W)
                if cols.size == 0:
                    continue
                bsum = beta[:, rows][:, :, cols].astype(np.float64)          # [K][h][w]
                gsum = gJ[:, rows][:, :, cols].astype(np.float64)            # [C][h][w]
                out[n] += np.einsum("k,khw,chw->c", basis[:, i, j].astype(np.float64), bsum, gsum)
    return out


def grad_tilt(J, tilt, g, coord_dtype=np.float64, absolute=False):
    """dL/dt [2][H][W] (fp64) of the warp out_c(p) = bilinear(J_c, p - t(p)) for a given blur J
    [C][H][W] and upstream g [C][H][W]: the derivative of the bilinear weights inside the cell,
    0 where the coordinate clamp is active. absolute=True returns the same sums over |terms|
    (the scale of their rounding error)."""
    J = np.asarray(J, np.float64)
    C_, H, W = J.shape
    g = np.asarray(g, np.float64)
    ya, yb, xa, xb, fy, fx, in_y, in_x = _warp_coords(tilt, H, W, coord_dtype)
    # d out / d sx = (1-fy)(J[ya][xb] - J[ya][xa]) + fy (J[yb][xb] - J[yb][xa]); sx = x - t_x
    if absolute:
        dsx = (1 - fy) * (abs(J[:, ya, xb]) + abs(J[:, ya, xa])) + fy * (abs(J[:, yb, xb]) + abs(J[:, yb, xa]))
        dsy = (1 - fx) * (abs(J[:, yb, xa]) + abs(J[:, ya, xa])) + fx * (abs(J[:, yb, xb]) + abs(J[:, ya, xb]))
        g = np.abs(g)
    else:
        dsx = (1 - fy) * (J[:, ya, xb] - J[:, ya, xa]) + fy * (J[:, yb, xb] - J[:, yb, xa])
        dsy = (1 - fx) * (J[:, yb, xa] - J[:, ya, xa]) + fx * (J[:, yb, xb] - J[:, ya, xb])
    sgn = 1.0 if absolute else -1.0
    gt = np.zeros((2, H, W))
    gt[0] = sgn * np.where(in_x, (g * dsx).sum(0), 0.0)
    gt[1] = sgn * np.where(in_y, (g * dsy).sum(0), 0.0)
    return gt


def backward(image, beta, tilt, basis, g, coord_dtype=np.float64):
    """(dL/dJ [C][H][W], dL/dbeta [K][H][W], dL/dt [2][H][W], dL/dI [C][H][W]) for upstream
    g [C][H][W]."""
    _, J, Ck = forward_from_beta(image, beta, tilt, basis)
    g = g.astype(np.float64)
    gJ = grad_J(tilt, g, coord_dtype)
    gbeta = np.einsum("chw,kchw->khw", gJ, Ck)
    gimage = grad_image(beta, basis, gJ)
    gt = grad_tilt(J, tilt, g, coord_dtype)
    return gJ, gbeta, gt, gimage


def backward_at(image, beta, tilt, basis, g, yx, coord_dtype=np.float64):
    """backward's dL/dbeta [n][K] and dL/dt [n][2] at the listed pixels only (full-size frames):
    dL/dJ over the whole frame (cheap), C_kc and J only where the listed pixels need them."""
    C_, H, W = image.shape
    g = g.astype(np.float64)
    gJ = grad_J(tilt, g, coord_dtype)
    ya, yb, xa, xb, fy, fx, in_y, in_x = _warp_coords(tilt, H, W, coord_dtype)
    gbeta = np.zeros((len(yx), beta.shape[0]))
    gt = np.zeros((len(yx), 2))
    for n, (y, x) in enumerate(yx):
        gbeta[n] = conv_at(image, basis, [(y, x)])[0] @ gJ[:, y, x]
        corners = [(ya[y, x], xa[y, x]), (ya[y, x], xb[y, x]), (yb[y, x], xa[y, x]), (yb[y, x], xb[y, x])]
        Ck = conv_at(image, basis, corners)                                  # [4][K][C]
        Jc = np.einsum("nk,nkc->nc", np.stack([beta[:, q, p] for q, p in corners]), Ck)  # J_c at corners
        j00, j01, j10, j11 = Jc
        a, b = fy[y, x], fx[y, x]
        dsx = (1 - a) * (j01 - j00) + a * (j11 - j10)
        dsy = (1 - b) * (j10 - j00) + b * (j11 - j01)
        gt[n, 0] = -(g[:, y, x] @ dsx) if in_x[y, x] else 0.0
        gt[n, 1] = -(g[:, y, x] @ dsy) if in_y[y, x] else 0.0
    return gbeta, gt


def _f16(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float64)


def mlp_preactivations(zernike, mlp, mask_precision="fp64"):
    """(pre1 [h1][H*W], pre2 [h2][H*W]) of one frame's MLP layers 1-2 (reading
    A11), fp64 values: "fp64" from exact operands; "fp16" from the fp16-rounded z, W1, W2 and a1
    the GPU multiplies (reading N5), biases exact."""
    z = np.asarray(zernike, np.float64)
    Z = z.reshape(z.shape[0], -1)
    b1, b2 = (np.asarray(mlp[k], np.float64) for k in ("b1", "b2"))
    if mask_precision == "fp16":
        pre1 = _f16(mlp["W1"]) @ _f16(Z.T.astype(np.float32)).T + b1[:, None]
        a1 = np.maximum(pre1, 0.0)
        pre2 = _f16(mlp["W2"]) @ _f16(a1.astype(np.float32)) + b2[:, None]
    else:
        W1, W2 = (np.asarray(mlp[k], np.float64) for k in ("W1", "W2"))
        pre1 = W1 @ Z + b1[:, None]
        pre2 = W2 @ np.maximum(pre1, 0.0) + b2[:, None]
    return pre1, pre2


def mlp_backward(zernike, gbeta, mlp, mask_precision="fp64", masks=None):
    """dL/dz [n_in][H][W] (fp64) of one frame through the P2S MLP (step a1, PAPER.md:280-283,
    reading A11: ReLU after layers 1-2, linear output), for dL/dbeta [K][H][W]:

        pre1 = W1 z + b1,  a1 = ReLU(pre1),  pre2 = W2 a1 + b2,  (beta = W3 ReLU(pre2) + b3)
        g2 = (W3^T dL/dbeta) [pre2 > 0],  g1 = (W2^T g2) [pre1 > 0],  dL/dz = W1^T g1

    The masks are integers decided by floats: mask_precision="fp16" decides them the way the GPU
    does (fp16-rounded z, weights and a1; reading N5), "fp64" from exact values (the
    finite-difference pins); masks=(m1 [h1][H*W], m2 [h2][H*W]) imposes them (the tests' check
    of the other valid answer where a pre-activation is within rounding of 0). The gradient
    values are fp64 either way."""
    z = np.asarray(zernike, np.float64)
    n_in, H, W = z.shape
    G3 = np.asarray(gbeta, np.float64).reshape(gbeta.shape[0], -1)
    W1, W2, W3 = (np.asarray(mlp[k], np.float64) for k in ("W1", "W2", "W3"))
    if masks is None:
        pre1, pre2 = mlp_preactivations(z, mlp, mask_precision)
        m1, m2 = pre1 > 0, pre2 > 0
    else:
        m1, m2 = masks
    g2 = (W3.T @ G3) * m2
    g1 = (W2.T @ g2) * m1
    return (W1.T @ g1).reshape(n_in, H, W)


def anchor_weights(n, G):
    """[n][G] fp64 matrix of the 1-D linear weights the anchor interpolation gives pixel index
    t (0..n-1) from anchor index a (reading N1: pixel centre t + 0.5,
    anchors at a n / (G - 1)): u = (t + 0.5)(G - 1)/n, i0 = min(floor(u), G - 2), weights
    1 - (u - i0) on i0 and u - i0 on i0 + 1; G = 1: all weight on the single anchor."""
    w = np.zeros((n, G))
    if G == 1:
        w[:, 0] = 1.0
        return w
    for t in range(n):
        u = (t + 0.5) * (G - 1) / n
        i0 = min(int(np.floor(u)), G - 2)
        f = u - i0
        w[t, i0] += 1.0 - f
        w[t, i0 + 1] += f
    return w


def anchors_backward(gfield, G):
    """dL/dA [B][n_in][G][G] (fp64) for dL/dz = gfield [B][n_in][H][W]: the transpose of the
    separable bilinear anchor interpolation z = Wy A Wx^T (per frame and mode), dL/dA = Wy^T dL/dz Wx."""
    g = np.asarray(gfield, np.float64)
    B, n_in, H, W = g.shape
    Wy, Wx = anchor_weights(H, G), anchor_weights(W, G)
    return np.einsum("ya,bkyx,xc->bkac", Wy, g, Wx)


def backward_color(image, zernike_c, tilt, basis, mlp, g, coord_dtype=np.float64, mask_precision="fp64"):
    """Adjoint of the wavelength-dependent colour render (oracle.render_color):
    channel c of a frame is a one-channel render with its own beta_c = P2S(z_c), so for one frame
    (image [C][H][W], zernike_c [C][n_in][H][W], tilt [2][H][W], g = dL/dout [C][H][W]):
        dL/dbeta_c = backward(I_c, beta_c, t, g_c).dbeta,   dL/dI_c = backward(...).dI,
        dL/dt = sum_c backward(...).dt,                       dL/dz_c = mlp_backward(z_c, dL/dbeta_c)
    Returns (dbeta [C][K][H][W], dt [2][H][W], dI [C][H][W], dz [C][n_in][H][W]), fp64."""
    from oracle import beta as _beta  # the C oracle's beta (forward of step a1)
    image = np.asarray(image)
    C = image.shape[0]
    gb, gi, gz = [], [], []
    gt = None
    for c in range(C):
        zc = np.ascontiguousarray(zernike_c[c], np.float32)
        bc = _beta(image[None, c:c + 1], zc[None], basis, mlp)[0]
        _, gbc, gtc, gic = backward(image[c:c + 1], bc, tilt, basis, g[c:c + 1], coord_dtype=coord_dtype)
        gb.append(gbc)
        gi.append(gic[0])
        gt = gtc if gt is None else gt + gtc
        gz.append(mlp_backward(zc.astype(np.float64), gbc, mlp, mask_precision))
    return np.stack(gb), gt, np.stack(gi), np.stack(gz)
