"""Pins of the CPU oracle against things other than itself (task rule ③).

Each test names the paper passage / DESIGN.md reading it pins and the independent source
of truth: a closed form, an invariant, brute force on tiny inputs, or a library routine
(torch nn.Linear, scipy.ndimage.convolve, torch conv2d, scipy.signal.fftconvolve,
torch grid_sample). None of them re-types the oracle's own loops. A plausible mistake in
the oracle — dropped term, wrong sign/index, transposed operand, correlation instead of
convolution, scatter instead of gather order, wrong boundary — fails at least one.
"""
import numpy as np
import pytest
import scipy.ndimage
import scipy.signal
import torch

import oracle
from paper_2107_11627_b200 import synth


def _mlp_const(n_in, h, K, b3):
    """W1..W3 = 0 => beta == b3 everywhere (spatially constant beta)."""
    return {"W1": np.zeros((h, n_in), np.float32), "b1": np.zeros(h, np.float32),
            "W2": np.zeros((h, h), np.float32), "b2": np.zeros(h, np.float32),
            "W3": np.zeros((K, h), np.float32), "b3": np.asarray(b3, np.float32)}


def _small(seed=0, B=1, C=1, H=24, W=20, K=6, S=5, n_in=7, h=9, tstd=1.3):
    spec = synth.custom("pin", 100 + seed, B=B, C=C, H=H, W=W, K=K, S=S, n_in=n_in, h1=h,
                        h2=h + 2, z_sigma=2.0, z_std=0.8, t_sigma=3.0, t_std=tstd)
    return synth.make_inputs(spec)


def _render(inp, tilt="same", **kw):
    t = inp.tilt if tilt == "same" else tilt
    return oracle.render(inp.image, inp.zernike, t, inp.basis, inp.mlp, want_blur=True, **kw)


# ---------------------------------------------------------------- step a1: P2S MLP
def test_mlp_matches_torch_linear_stack():
    """P6 — PAPER.md:283 'three fully connected layers' (ReLU hidden, linear out, A11)
    vs torch.nn.Linear/ReLU in float64 (library routine)."""
    inp = _small(1)
    b = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)
    m = inp.mlp
    net = torch.nn.Sequential(torch.nn.Linear(*m["W1"].shape[::-1]), torch.nn.ReLU(),
                              torch.nn.Linear(*m["W2"].shape[::-1]), torch.nn.ReLU(),
                              torch.nn.Linear(*m["W3"].shape[::-1])).double()
    with torch.no_grad():
        for li, layer in zip((1, 2, 3), (net[0], net[2], net[4])):
            layer.weight.copy_(torch.from_numpy(m[f"W{li}"].astype(np.float64)))
            layer.bias.copy_(torch.from_numpy(m[f"b{li}"].astype(np.float64)))
        z = torch.from_numpy(inp.zernike[0].astype(np.float64)).permute(1, 2, 0)  # H W n_in
        ref = net(z).permute(2, 0, 1).numpy()
    np.testing.assert_allclose(b[0], ref, rtol=0, atol=1e-12)
    # the stack must be non-trivial: some hidden units clipped, output not affine in z
    assert np.std(ref) > 0.05


def test_mlp_zero_weights_gives_bias():
    """S:272 idea — zero weights => output equals b3 (no output activation, A11)."""
    inp = _small(2)
    K = inp.basis.shape[0]
    b3 = np.linspace(-1, 1, K).astype(np.float32)
    mlp = _mlp_const(inp.zernike.shape[1], 9, K, b3)
    mlp["W2"] = np.zeros((9, 9), np.float32)
    b = oracle.beta(inp.image, inp.zernike, inp.basis, mlp)
    np.testing.assert_array_equal(b[0], np.broadcast_to(b3[:, None, None], b[0].shape))


# ---------------------------------------------------------------- step a2: Eq. (5)
def test_identity_delta_basis():
    """North-star (a): K=1, phi = centred Dirac, beta = 1 => J = I and out = I (zero tilt)."""
    for S in (1, 15):
        inp = _small(3, S=S, K=1, tstd=0.0)
        basis = np.zeros((1, S, S), np.float32)
        basis[0, S // 2, S // 2] = 1.0
        inp.basis = basis
        inp.mlp = _mlp_const(inp.zernike.shape[1], 4, 1, [1.0])
        out, J = _render(inp)
        np.testing.assert_array_equal(J, inp.image.astype(np.float64))
        np.testing.assert_array_equal(out, inp.image.astype(np.float64))


def test_delta_basis_shift_sign():
    """P8 — true convolution (A2, A3): phi[r+dy][r+dx] = 1 moves content by +(dy, dx),
    replicate boundary (A4): J(y,x) = I[clamp(y-dy)][clamp(x-dx)]."""
    S, r = 7, 3
    for dy, dx in ((2, -1), (-3, 3), (0, 1)):
        inp = _small(4, S=S, K=1, tstd=0.0)
        basis = np.zeros((1, S, S), np.float32)
        basis[0, r + dy, r + dx] = 1.0
        inp.basis = basis
        inp.mlp = _mlp_const(inp.zernike.shape[1], 4, 1, [1.0])
        _, J = _render(inp)
        H, W = inp.image.shape[2:]
        yy = np.clip(np.arange(H) - dy, 0, H - 1)
        xx = np.clip(np.arange(W) - dx, 0, W - 1)
        np.testing.assert_array_equal(J[0, 0], inp.image[0, 0][yy][:, xx].astype(np.float64))


def test_constant_beta_equals_scipy_and_torch_conv():
    """P2 — spatially constant beta: J = I * (sum_k beta0_k phi_k) equals
    scipy.ndimage.convolve(mode='nearest') and torch conv2d(replicate pad, flipped taps)."""
    inp = _small(5, C=3, S=9, K=5, H=30, W=17, tstd=0.0)
    beta0 = np.array([0.7, -0.4, 1.3, 0.2, -0.9], np.float32)
    inp.mlp = _mlp_const(inp.zernike.shape[1], 6, 5, beta0)
    _, J = _render(inp)
    h = np.tensordot(beta0.astype(np.float64), inp.basis.astype(np.float64), axes=1)
    for c in range(3):
        ref = scipy.ndimage.convolve(inp.image[0, c].astype(np.float64), h, mode="nearest")
        np.testing.assert_allclose(J[0, c], ref, rtol=0, atol=1e-12)
    x = torch.from_numpy(inp.image.astype(np.float64))
    xp = torch.nn.functional.pad(x, (4, 4, 4, 4), mode="replicate")
    w = torch.from_numpy(np.flip(h, (0, 1)).copy())[None, None].repeat(3, 1, 1, 1)
    ref_t = torch.nn.functional.conv2d(xp, w, groups=3).numpy()
    np.testing.assert_allclose(J, ref_t, rtol=0, atol=1e-12)


def test_one_hot_beta_each_basis():
    """P5 — beta = e_k => J = I * phi_k (per-k indexing), FFT convolution on an
    edge-padded image (scipy.signal.fftconvolve, 'valid')."""
    inp = _small(6, S=7, K=4, H=21, W=26, tstd=0.0)
    I = inp.image[0, 0].astype(np.float64)
    Ip = np.pad(I, 3, mode="edge")
    for k in range(4):
        e = np.zeros(4, np.float32)
        e[k] = 1
        inp.mlp = _mlp_const(inp.zernike.shape[1], 5, 4, e)
        _, J = _render(inp)
        ref = scipy.signal.fftconvolve(Ip, inp.basis[k].astype(np.float64), mode="valid")
        np.testing.assert_allclose(J[0, 0], ref, rtol=0, atol=1e-12)


def test_brute_force_spatially_varying_conv():
    """North-star (c) — Eq. (3)/(4): per-pixel PSF
    h_{y,x} = sum_k beta_k(y,x) phi_k applied directly equals the Eq. (5) basis-sum form."""
    inp = _small(7, C=2, S=5, K=6, H=13, W=11)
    _, J = _render(inp, tilt=None)
    beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)[0]  # K H W (pinned by P6)
    H, W, S, r = 13, 11, 5, 2
    phi = inp.basis.astype(np.float64)
    for c in range(2):
        I = inp.image[0, c].astype(np.float64)
        ref = np.zeros((H, W))
        for y in range(H):
            for x in range(W):
                h = np.tensordot(beta[:, y, x], phi, axes=1)       # the row h_n of H (Eq. 3)
                for i in range(S):
                    for j in range(S):
                        ref[y, x] += h[i, j] * I[min(max(y - (i - r), 0), H - 1),
                                                 min(max(x - (j - r), 0), W - 1)]
        np.testing.assert_allclose(J[0, c], ref, rtol=0, atol=1e-12)


def test_gather_order_delta_image():
    """P1 / reading A1 — Eq. (5) weights at the OUTPUT pixel: for a delta image at p0,
    J(p) = sum_k beta_k(p) phi_k(p - p0) (gather). The scatter order
    sum_k (beta_k I) * phi_k would give beta_k(p0) instead and must differ."""
    inp = _small(8, S=7, K=5, H=20, W=20, tstd=0.0)
    I = np.zeros((20, 20), np.float32)
    I[10, 9] = 1.0
    inp.image = I[None, None]
    _, J = _render(inp)
    beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)[0]
    ref = np.zeros((20, 20))
    scat = np.zeros((20, 20))
    for y in range(20):
        for x in range(20):
            i, j = y - 10 + 3, x - 9 + 3
            if 0 <= i < 7 and 0 <= j < 7:
                ref[y, x] = np.dot(beta[:, y, x], inp.basis[:, i, j].astype(np.float64))
                scat[y, x] = np.dot(beta[:, 10, 9], inp.basis[:, i, j].astype(np.float64))
    np.testing.assert_allclose(J[0, 0], ref, rtol=0, atol=1e-13)
    assert np.abs(ref - scat).max() > 1e-2


def test_mean_preservation_constant_image():
    """North-star (d): W = 0, b3 = s/|s|^2 with s_k = sum of taps of phi_k => sum_k beta_k s_k = 1;
    a constant image stays constant through the blur (replicate) and any warp."""
    inp = _small(9, C=3, S=9, K=7, tstd=2.5)
    s = inp.basis.astype(np.float64).sum(axis=(1, 2))
    inp.mlp = _mlp_const(inp.zernike.shape[1], 5, 7, (s / np.dot(s, s)).astype(np.float32))
    inp.image = np.full_like(inp.image, 0.625)
    out, J = _render(inp)
    b3 = inp.mlp["b3"].astype(np.float64)
    expect = 0.625 * np.dot(b3, s)  # = 0.625 up to the fp32 rounding of b3
    assert abs(np.dot(b3, s) - 1) < 1e-6
    np.testing.assert_allclose(J, expect, rtol=0, atol=1e-13)
    np.testing.assert_allclose(out, expect, rtol=0, atol=1e-13)


def test_linearity_in_image():
    """North-star (b): out(2*I1 - I2) = 2*out(I1) - out(I2) with fixed Z and tilt (A12: no clamp).
    Images on a 2^-10 grid so the fp32 combination is exact."""
    inp = _small(10, C=2, S=5, K=4)
    rng = np.random.default_rng(0)
    I1 = (rng.integers(0, 1024, inp.image.shape) / 1024).astype(np.float32)
    I2 = (rng.integers(0, 1024, inp.image.shape) / 1024).astype(np.float32)
    outs = []
    for I in (I1, I2, 2 * I1 - I2):
        inp.image = I
        outs.append(_render(inp)[0])
    lhs, rhs = outs[2], 2 * outs[0] - outs[1]
    assert np.abs(lhs - rhs).max() <= 1e-12 * max(1.0, np.abs(lhs).max())


def test_colour_channels_share_beta():
    """P7 / A13: a gray image replicated to 3 channels gives 3 identical outputs."""
    inp = _small(11, C=3, S=5, K=4)
    inp.image = np.repeat(inp.image[:, :1], 3, axis=1)
    out, J = _render(inp)
    assert np.array_equal(out[0, 0], out[0, 1]) and np.array_equal(out[0, 0], out[0, 2])


# ---------------------------------------------------------------- step a3: tilt warp
def test_zero_tilt_is_identity_warp():
    """North-star (e): t = 0 => out = J exactly."""
    inp = _small(12, C=2, tstd=0.0)
    out, J = _render(inp)
    np.testing.assert_array_equal(out, J)


def test_warp_matches_grid_sample():
    """P3 — backward bilinear warp, clamp-to-edge (A6-A8) equals torch grid_sample
    (bilinear, padding 'border', align_corners=True) with grid = p - t normalised."""
    rng = np.random.default_rng(1)
    B, C, H, W = 2, 3, 19, 23
    J = rng.standard_normal((B, C, H, W))
    t = (rng.standard_normal((B, 2, H, W)) * 3).astype(np.float32)
    out = oracle.warp(J, t)
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    gx = 2 * (xx[None] - t[:, 0].astype(np.float64)) / (W - 1) - 1
    gy = 2 * (yy[None] - t[:, 1].astype(np.float64)) / (H - 1) - 1
    grid = torch.from_numpy(np.stack([gx, gy], -1))
    ref = torch.nn.functional.grid_sample(torch.from_numpy(J), grid, mode="bilinear",
                                          padding_mode="border", align_corners=True).numpy()
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)


def test_warp_integer_and_half_shift():
    """P4: t = (1, 0) moves content right one pixel, column 0 replicated;
    t = (0.5, 0) averages with the left neighbour. t = (0, -2): content moves up 2 rows."""
    rng = np.random.default_rng(2)
    J = rng.standard_normal((1, 1, 8, 9))
    t = np.zeros((1, 2, 8, 9), np.float32)
    t[:, 0] = 1.0
    left = J[..., np.maximum(np.arange(9) - 1, 0)]
    np.testing.assert_array_equal(oracle.warp(J, t), left)
    t[:, 0] = 0.5
    np.testing.assert_allclose(oracle.warp(J, t), 0.5 * (left + J), rtol=0, atol=1e-15)
    t[:, 0] = 0.0
    t[:, 1] = -2.0
    np.testing.assert_array_equal(oracle.warp(J, t), J[..., np.minimum(np.arange(8) + 2, 7), :])


def test_warp_reproduces_affine_field():
    """Bilinear interpolation is exact on affine functions: for J = a + b*y + c*x and samples
    that stay inside the image, out(y,x) = a + b*(y - t1) + c*(x - t0)."""
    H, W = 16, 18
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    J = (0.3 + 0.7 * yy - 1.1 * xx)[None, None].astype(np.float64)
    rng = np.random.default_rng(3)
    t = rng.uniform(-0.9, 0.9, (1, 2, H, W)).astype(np.float32)
    out = oracle.warp(J, t)
    ref = 0.3 + 0.7 * (yy - t[0, 1].astype(np.float64)) - 1.1 * (xx - t[0, 0].astype(np.float64))
    inner = (slice(1, H - 1), slice(1, W - 1))
    np.testing.assert_allclose(out[0, 0][inner], ref[inner], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- sampled / banded paths
def test_pixels_and_rows_agree_with_full_render():
    """The sampled path (used for full-size GPU parity) and the row-band path (used for the
    bounded cpu_baseline sample) compute exactly what the full render computes."""
    inp = _small(13, B=2, C=3, S=7, K=5, H=22, W=19, tstd=2.0)
    out, J = _render(inp)
    rng = np.random.default_rng(4)
    bxy = np.stack([rng.integers(0, 2, 40), rng.integers(0, 22, 40), rng.integers(0, 19, 40)], 1)
    bxy[:4] = [[0, 0, 0], [1, 21, 18], [0, 0, 18], [1, 21, 0]]
    Jp, op = oracle.pixels(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, bxy)
    np.testing.assert_array_equal(Jp, J[bxy[:, 0], :, bxy[:, 1], bxy[:, 2]])
    np.testing.assert_array_equal(op, out[bxy[:, 0], :, bxy[:, 1], bxy[:, 2]])
    out_band, _ = oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, rows=(5, 12))
    np.testing.assert_array_equal(out_band[:, :, 5:12], out[:, :, 5:12])


def test_thread_count_does_not_change_results():
    """Determinism regardless of worker count."""
    inp = _small(14, C=2, S=5, K=4)
    a, _ = oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, threads=1)
    b, _ = oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, threads=5)
    np.testing.assert_array_equal(a, b)


# ---- anchor grid -> dense Zernike field (Sec. 3.4;
#      registration: DESIGN.md reading N1 — pixel centres at (y + 0.5, x + 0.5), anchors spanning
#      the image corner to corner at (i H/(G-1), j W/(G-1)))

def _anchor_coords(G, H, W):
    return np.arange(G) * H / (G - 1), np.arange(G) * W / (G - 1)


def test_anchor_interp_constant_and_single_anchor():
    """Constant anchors give a constant field; G = 1 is a constant field (closed forms)."""
    a = np.full((2, 3, 5, 5), 0.375, np.float32)
    np.testing.assert_allclose(oracle.interp_anchors(a, 17, 23), 0.375, rtol=0, atol=1e-15)  # fp64 weights
    a1 = np.array([[[[1.25]], [[-0.5]]]], np.float32)
    f1 = oracle.interp_anchors(a1, 7, 9)
    assert np.array_equal(f1[0, 0], np.full((7, 9), 1.25)) and np.array_equal(f1[0, 1], np.full((7, 9), -0.5))


@pytest.mark.parametrize("G,H,W", [(2, 8, 8), (5, 37, 21), (16, 64, 96), (9, 512, 200)])
def test_anchor_interp_reproduces_bilinear_functions(G, H, W):
    """Bilinear interpolation reproduces any function a + b u + c v + d u v exactly, so with
    anchors sampled from one the field must equal it at the pixel centres (y+0.5, x+0.5): a
    shifted or scaled registration, a swapped axis or a wrong weight fails."""
    u, v = _anchor_coords(G, H, W)
    co = (0.25, -0.125, 0.0625, 0.001953125)  # dyadic: exact in fp32
    f = lambda uu, vv: co[0] + co[1] * uu + co[2] * vv + co[3] * uu * vv  # noqa: E731
    A = f(u[:, None], v[None, :]).astype(np.float32)[None, None]
    yc, xc = np.arange(H) + 0.5, np.arange(W) + 0.5
    ref = f(yc[:, None], xc[None, :])
    got = oracle.interp_anchors(A.astype(np.float64).astype(np.float32), H, W)[0, 0]
    # the anchors themselves are fp32-rounded samples of f: compare against interpolating those
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5 * (1 + np.abs(ref).max()))


def test_anchor_interp_matches_scipy_regular_grid():
    """Random anchors: equals scipy.interpolate.RegularGridInterpolator(linear) on the anchor
    coordinates, evaluated at the pixel centres (library routine)."""
    from scipy.interpolate import RegularGridInterpolator
    rng = np.random.default_rng(7)
    G, H, W = 6, 41, 29
    A = rng.standard_normal((1, 4, G, G)).astype(np.float32)
    got = oracle.interp_anchors(A, H, W)
    u, v = _anchor_coords(G, H, W)
    yy, xx = np.meshgrid(np.arange(H) + 0.5, np.arange(W) + 0.5, indexing="ij")
    for k in range(4):
        ref = RegularGridInterpolator((u, v), A[0, k].astype(np.float64))(np.stack([yy, xx], -1))
        np.testing.assert_allclose(got[0, k], ref, rtol=0, atol=1e-12)


def test_anchor_interp_exact_at_anchor_pixels():
    """Where an anchor coincides with a pixel centre (H = W = 3, G = 3: anchor 1 at 1.5) the field
    takes that anchor's value exactly (SPEC S:347 example)."""
    A = np.arange(9, dtype=np.float32).reshape(1, 1, 3, 3) * 0.5 - 1.0
    f = oracle.interp_anchors(A, 3, 3)
    assert f[0, 0, 1, 1] == A[0, 0, 1, 1]


# ---- correlated anchor sampling (stand-in covariance:
#      DESIGN.md reading N3) — oracle/sampler.py

def test_philox_known_answers():
    """Philox4x32-10 reproduces the Random123 known-answer vectors (Salmon et al., SC'11)."""
    from oracle import sampler
    out = sampler.philox4x32_10([[0, 0, 0, 0], [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344]],
                                [[0, 0], [0xa4093822, 0x299f31d0]])
    assert [int(v) for v in out[0]] == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert [int(v) for v in out[1]] == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_sampler_normals_are_standard_normal():
    """Box-Muller on Philox words: mean 0, variance 1, Kolmogorov-Smirnov vs N(0,1)."""
    import scipy.stats
    from oracle import sampler
    z = np.concatenate([sampler.normals(1234, f, 64, 33).ravel() for f in range(4)])  # 540k draws
    n = z.size
    assert abs(z.mean()) < 5 / np.sqrt(n)
    assert abs(z.var() - 1) < 5 * np.sqrt(2 / n)
    assert scipy.stats.kstest(z, "norm").pvalue > 1e-3
    # different frames / seeds give different streams
    assert not np.allclose(sampler.normals(1234, 0, 4, 3), sampler.normals(1234, 1, 4, 3))
    assert not np.allclose(sampler.normals(1234, 0, 4, 3), sampler.normals(1235, 0, 4, 3))


def test_sampler_identity_covariance_returns_the_normals():
    """corr_len 0 (s = identity up to the 1e-6 jitter) and R = I: the anchors are z itself."""
    from oracle import sampler
    A = sampler.sample(7, 3, 2, 5, 4, corr_len=0.0, mode_cov=np.eye(4))
    for f in range(2):
        z = sampler.normals(7, 3 + f, 5, 4).reshape(5, 5, 4).transpose(2, 0, 1)
        np.testing.assert_allclose(A[f], z * (1 + 1e-6), rtol=1e-12, atol=1e-12)  # two spatial factors


def test_sampler_empirical_covariance():
    """Across many frames the anchors' covariance is R (x) s (x) s (Monte-Carlo, 4000 frames)."""
    from oracle import sampler
    G, n_in, L = 3, 2, 1.5
    rng = np.random.default_rng(3)
    M = rng.standard_normal((n_in, n_in))
    R = M @ M.T / n_in + 0.5 * np.eye(n_in)
    A = sampler.sample(99, 0, 4000, G, n_in, corr_len=L, mode_cov=R).reshape(4000, -1)
    emp = A.T @ A / A.shape[0]
    s = sampler.spatial_cov(G, L)
    ref = np.kron(R, np.kron(s, s))
    assert np.abs(emp - ref).max() < 6 * np.sqrt(2 / 4000) * np.abs(ref).max()


def test_dense_sampler_reduces_to_the_separable_one():
    """A dense spatial correlation equal to s (x) s (the separable stand-in written out) gives the
    separable sampler's anchors: the Kronecker product of the Cholesky factors is the Cholesky
    factor of the Kronecker product (both lower triangular with a positive diagonal)."""
    from oracle import sampler
    rng = np.random.default_rng(5)
    M = rng.standard_normal((3, 3))
    R = M @ M.T / 3 + 0.3 * np.eye(3)
    for G, L in ((1, 0.0), (4, 1.5), (6, 0.0), (7, 2.5)):
        sep = sampler.sample(11, 2, 3, G, 3, corr_len=L, mode_cov=R)
        den = sampler.sample_dense(11, 2, 3, G, 3, synth.anchor_cov_separable(G, L), mode_cov=R)
        # (equal up to rounding amplified by the condition number: the Gaussian s with a 1e-6
        # jitter has cond ~ 1e6, so the two factorisations agree to ~1e-9)
        np.testing.assert_allclose(den, sep, rtol=0, atol=1e-7)
        # the factor passed directly (is_factor) is the same draw
        Lf = np.linalg.cholesky(synth.anchor_cov_separable(G, L))
        Lf_up = Lf + np.triu(np.ones_like(Lf), 1) * 7.0  # upper part ignored
        np.testing.assert_allclose(sampler.sample_dense(11, 2, 3, G, 3, Lf_up, mode_cov=R, is_factor=True), den,
                                   rtol=0, atol=1e-12)


def test_dense_sampler_empirical_covariance_nonseparable():
    """Across 4000 frames the anchors' covariance is R (x) C for the NON-separable exponential
    correlation C (Monte-Carlo), which no Kronecker-factored sampler can produce."""
    from oracle import sampler
    G, n_in = 3, 2
    rng = np.random.default_rng(4)
    M = rng.standard_normal((n_in, n_in))
    R = M @ M.T / n_in + 0.5 * np.eye(n_in)
    Cs = synth.anchor_cov_exp(G, 1.2)
    # C is not separable: it differs from the Kronecker product of its own row/column marginals
    assert np.abs(Cs - np.kron(Cs[::G, ::G], Cs[:G, :G])).max() > 1e-2
    A = sampler.sample_dense(99, 0, 4000, G, n_in, Cs, mode_cov=R).reshape(4000, -1)
    emp = A.T @ A / A.shape[0]
    ref = np.kron(R, Cs)
    assert np.abs(emp - ref).max() < 6 * np.sqrt(2 / 4000) * np.abs(ref).max()
    assert np.all(np.linalg.eigvalsh(synth.anchor_cov_exp(8, 3.0)) > 0)  # positive definite at G = 8


@pytest.mark.parametrize("shape", [dict(B=1, C=3, H=9, W=11, K=4, S=5), dict(B=2, C=1, H=6, W=5, K=3, S=7),
                                   dict(B=1, C=2, H=1, W=1, K=2, S=3), dict(B=1, C=1, H=4, W=13, K=1, S=1)])
def test_c_adjoint_blur_matches_numpy_adjoint(shape):
    """The C oracle's adjoint of Eq. 5 (dL/dbeta, dL/dI: the whole-frame reference of the GPU's
    cfg3 adjoint) equals oracle/adjoint.py's (pinned above by central finite differences)."""
    from oracle import adjoint
    rng = np.random.default_rng(sum(shape.values()))
    B, C, H, W, K, S = (shape[k] for k in "BCHWKS")
    image = rng.random((B, C, H, W)).astype(np.float32)
    basis = rng.standard_normal((K, S, S)).astype(np.float32)
    beta = rng.standard_normal((B, K, H, W))
    gJ = rng.standard_normal((B, C, H, W))
    gb, gi = oracle.adjoint_blur(image, basis, beta, gJ, threads=3)
    for b in range(B):
        Ck = adjoint.conv_all(image[b], basis)
        np.testing.assert_allclose(gb[b], np.einsum("chw,kchw->khw", gJ[b], Ck), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(gi[b], adjoint.grad_image(beta[b], basis, gJ[b]), rtol=1e-12, atol=1e-12)


def test_c_adjoint_blur_dot_product_identities():
    """<dL/dJ, J> = <dL/dbeta, beta> = <dL/dI, I> with J the C oracle's own forward blur (J is
    linear in I and in beta for fixed beta / I), on a ragged 3-channel frame with replicate borders."""
    spec = synth.custom("adjid", 321, B=1, C=3, H=21, W=34, K=6, S=9, h1=16, h2=16, t_std=0.0)
    inp = synth.make_inputs(spec)
    beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)
    _, J = oracle.render(inp.image, inp.zernike, None, inp.basis, inp.mlp, want_blur=True)
    gJ = np.random.default_rng(8).standard_normal(J.shape)
    gb, gi = oracle.adjoint_blur(inp.image, inp.basis, beta, gJ)
    lhs = float((gJ * J).sum())
    assert abs(lhs - float((gb * beta).sum())) <= 1e-10 * np.abs(gJ * J).sum()
    assert abs(lhs - float((gi * inp.image).sum())) <= 1e-10 * np.abs(gJ * J).sum()


# ---- adjoint of steps a2-a3 ("differentiable module") —
#      oracle/adjoint.py, pinned by finite differences of its independent forward

def _adj_problem(seed=0, C=2, H=5, W=7, K=3, S=3, t_std=0.8):
    rng = np.random.default_rng(seed)
    image = rng.random((C, H, W))
    basis = rng.standard_normal((K, S, S))
    beta = rng.standard_normal((K, H, W))
    tilt = t_std * rng.standard_normal((2, H, W))
    g = rng.standard_normal((C, H, W))
    return image, basis, beta, tilt, g


def test_adjoint_beta_matches_finite_differences():
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(1)
    _, gbeta, _, _ = adjoint.backward(image, beta, tilt, basis, g)
    rng = np.random.default_rng(2)
    for _ in range(12):
        k, y, x = rng.integers(0, beta.shape[0]), rng.integers(0, beta.shape[1]), rng.integers(0, beta.shape[2])
        e = np.zeros_like(beta)
        e[k, y, x] = 1e-3
        lp = np.sum(g * adjoint.forward_from_beta(image, beta + e, tilt, basis)[0])
        lm = np.sum(g * adjoint.forward_from_beta(image, beta - e, tilt, basis)[0])
        assert abs((lp - lm) / 2e-3 - gbeta[k, y, x]) < 1e-9 * (1 + abs(gbeta[k, y, x]))  # linear in beta


def test_adjoint_tilt_matches_finite_differences():
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(3, t_std=1.3)
    _, _, gt, _ = adjoint.backward(image, beta, tilt, basis, g)
    rng = np.random.default_rng(4)
    for _ in range(16):
        ch, y, x = rng.integers(0, 2), rng.integers(0, tilt.shape[1]), rng.integers(0, tilt.shape[2])
        e = np.zeros_like(tilt)
        e[ch, y, x] = 1e-7
        lp = np.sum(g * adjoint.forward_from_beta(image, beta, tilt + e, basis)[0])
        lm = np.sum(g * adjoint.forward_from_beta(image, beta, tilt - e, basis)[0])
        assert abs((lp - lm) / 2e-7 - gt[ch, y, x]) < 1e-5 * (1 + abs(gt[ch, y, x]))


def test_adjoint_warp_dot_product_identity():
    """<g, warp(J)> = <dL/dJ, J>: the scattered bilinear weights are the exact transpose."""
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(5, H=9, W=11, t_std=2.5)  # tilts reach the clamp
    out, J, _ = adjoint.forward_from_beta(image, beta, tilt, basis)
    gJ, _, _, _ = adjoint.backward(image, beta, tilt, basis, g)
    assert abs(np.sum(g * out) - np.sum(gJ * J)) < 1e-10 * np.sum(np.abs(g * out))


def test_adjoint_forward_matches_render_oracle():
    """forward_from_beta with the MLP's beta reproduces p2s_oracle_render (two independent codes)."""
    from oracle import adjoint
    spec = synth.custom("adjf", 401, B=1, C=2, H=6, W=9, K=5, S=5, h1=16, h2=16, t_std=1.2)
    inp = synth.make_inputs(spec)
    beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)[0]
    out, J, _ = adjoint.forward_from_beta(inp.image[0], beta, inp.tilt[0], inp.basis)
    ref, Jref = oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, want_blur=True)
    np.testing.assert_allclose(J, Jref[0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out, ref[0], rtol=0, atol=1e-12)


def test_adjoint_conv_at_brute_force():
    """conv_at (the sampled-pixel form the full-size GPU test uses) == the convolution written as
    four nested loops over the definition, and == conv_all at the same pixels."""
    from oracle import adjoint
    rng = np.random.default_rng(6)
    C, H, W, K, S = 2, 6, 8, 3, 5
    image, basis = rng.random((C, H, W)), rng.standard_normal((K, S, S))
    r = S // 2
    yx = [(0, 0), (H - 1, W - 1), (2, 3), (5, 0), (0, 7)]
    got = adjoint.conv_at(image, basis, yx)
    full = adjoint.conv_all(image, basis)
    for n, (y, x) in enumerate(yx):
        for k in range(K):
            for c in range(C):
                ref = 0.0
                for i in range(S):
                    for j in range(S):
                        yy = min(max(y - (i - r), 0), H - 1)
                        xx = min(max(x - (j - r), 0), W - 1)
                        ref += basis[k, i, j] * image[c, yy, xx]
                assert abs(got[n, k, c] - ref) < 1e-12
                assert abs(full[k, c, y, x] - ref) < 1e-12


def test_adjoint_backward_at_matches_backward():
    """The sampled-pixel form agrees with the whole-frame backward (pinned above by finite
    differences), clamp-active pixels included."""
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(7, H=9, W=11, t_std=2.5)
    _, gbeta, gt, _ = adjoint.backward(image, beta, tilt, basis, g)
    yx = [(y, x) for y in range(9) for x in range(11)]
    gb_at, gt_at = adjoint.backward_at(image, beta, tilt, basis, g, yx)
    ys, xs = np.array(yx).T
    np.testing.assert_allclose(gb_at, gbeta[:, ys, xs].T, rtol=0, atol=1e-11)
    np.testing.assert_allclose(gt_at, gt[:, ys, xs].T, rtol=0, atol=1e-11)


def test_adjoint_fp32_cells_agree_away_from_cell_edges():
    """coord_dtype=float32 only moves the cell decision: where fp64 and fp32 s = p - t pick the
    same cell, dL/dt and dL/dJ agree to fp32 rounding of s."""
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(8, H=9, W=11, t_std=2.5)
    tilt = tilt.astype(np.float32)
    gJ64, gb64, gt64, _ = adjoint.backward(image, beta, tilt, basis, g)
    gJ32, gb32, gt32, _ = adjoint.backward(image, beta, tilt, basis, g, coord_dtype=np.float32)
    c64 = adjoint._warp_coords(tilt, 9, 11)
    c32 = adjoint._warp_coords(tilt, 9, 11, np.float32)
    same = np.all([np.array_equal(a, b) for a, b in zip(c64[:4], c32[:4])])
    assert same  # no fp32/fp64 cell flips on this problem: the two forms must then agree
    np.testing.assert_allclose(gt32, gt64, rtol=0, atol=1e-5 * (1 + np.abs(gt64).max()))
    np.testing.assert_allclose(gJ32, gJ64, rtol=0, atol=1e-5 * (1 + np.abs(gJ64).max()))



def test_adjoint_image_matches_finite_differences():
    """dL/dI by central differences of the forward (J is linear in I: differences are exact up to
    rounding), borders and corners included (S = 5 on a 5x7 frame: every pixel is near one)."""
    from oracle import adjoint
    image, basis, beta, tilt, g = _adj_problem(9, K=3, S=5)
    *_, gI = adjoint.backward(image, beta, tilt, basis, g)
    C, H, W = image.shape
    for c in range(C):
        for y in range(H):
            for x in range(W):
                e = np.zeros_like(image)
                e[c, y, x] = 1e-3
                lp = np.sum(g * adjoint.forward_from_beta(image + e, beta, tilt, basis)[0])
                lm = np.sum(g * adjoint.forward_from_beta(image - e, beta, tilt, basis)[0])
                assert abs((lp - lm) / 2e-3 - gI[c, y, x]) < 1e-9 * (1 + abs(gI[c, y, x]))


def test_adjoint_image_dot_product_and_sampled_form():
    """<dL/dJ, J(I)> = <dL/dI, I> (J is linear in I), and grad_image_at (per-pixel preimage
    rectangles, the full-size GPU test's form) == grad_image at every pixel, S > frame included."""
    from oracle import adjoint
    for seed, H, W, S in ((10, 9, 11, 5), (11, 6, 4, 9)):
        image, basis, beta, tilt, g = _adj_problem(seed, H=H, W=W, K=4, S=S)
        gJ, _, _, gI = adjoint.backward(image, beta, tilt, basis, g)
        _, J, _ = adjoint.forward_from_beta(image, beta, tilt, basis)
        assert abs(np.sum(gJ * J) - np.sum(gI * image)) < 1e-10 * np.sum(np.abs(gJ * J))
        yx = [(y, x) for y in range(H) for x in range(W)]
        at = adjoint.grad_image_at(beta, basis, gJ, yx)
        ys, xs = np.array(yx).T
        np.testing.assert_allclose(at, gI[:, ys, xs].T, rtol=0, atol=1e-11)


# ---- wavelength-dependent colour

def test_render_color_reduces_to_shared_beta():
    """One Zernike field for every channel (the paper's 'simulate the RGB channels identically',
    P:320, reading A13) makes render_color == render exactly; and channel c of render_color
    depends only on channel c's field (swapping another channel's field leaves it unchanged)."""
    spec = synth.custom("col", 501, B=2, C=3, H=7, W=9, K=5, S=5, h1=16, h2=16, t_std=1.2)
    inp = synth.make_inputs(spec)
    same = np.repeat(inp.zernike[:, None], 3, axis=1)
    o1, J1 = oracle.render_color(inp.image, same, inp.tilt, inp.basis, inp.mlp, want_blur=True)
    o0, J0 = oracle.render(inp.image, inp.zernike, inp.tilt, inp.basis, inp.mlp, want_blur=True)
    np.testing.assert_array_equal(o1, o0)
    np.testing.assert_array_equal(J1, J0)
    other = same.copy()
    other[:, 2] = 1.7 * same[:, 2] + 0.3
    o2, _ = oracle.render_color(inp.image, other, inp.tilt, inp.basis, inp.mlp)
    np.testing.assert_array_equal(o2[:, :2], o0[:, :2])
    assert np.abs(o2[:, 2] - o0[:, 2]).max() > 1e-3


def test_mlp_backward_matches_finite_differences():
    """dL/dz through the P2S MLP: central differences of the C oracle's beta (an independent
    forward) for L = <g, beta(z)>; and the fp16-mask form equals the exact one when no
    pre-activation is near zero (checked on this input)."""
    from oracle import adjoint
    spec = synth.custom("mlpb", 402, B=1, C=1, H=3, W=4, K=6, S=3, h1=12, h2=10)
    inp = synth.make_inputs(spec)
    z = inp.zernike.astype(np.float64)
    g = np.random.default_rng(3).standard_normal((6, 3, 4))
    dz = adjoint.mlp_backward(z[0], g, inp.mlp)
    loss = lambda zz: np.sum(g * oracle.beta(inp.image, zz.astype(np.float32), inp.basis, inp.mlp)[0])  # noqa: E731
    rng = np.random.default_rng(4)
    for _ in range(10):
        i, y, x = rng.integers(0, z.shape[1]), rng.integers(0, 3), rng.integers(0, 4)
        e = np.zeros_like(z)
        e[0, i, y, x] = 1e-2   # fp32 inputs to the oracle: a step well above their rounding
        fd = (loss(z + e) - loss(z - e)) / 2e-2
        assert abs(fd - dz[i, y, x]) < 1e-4 * (1 + abs(dz[i, y, x])), (fd, dz[i, y, x])
    # masks decided in fp16 agree here (no pre-activation within rounding of 0)
    np.testing.assert_allclose(adjoint.mlp_backward(z[0], g, inp.mlp, "fp16"), dz, rtol=0, atol=1e-12)


def test_mlp_preactivations_reproduce_c_oracle_beta():
    """The layer-1/2 pre-activations the dL/dz masks are decided on: W3 ReLU(pre2) + b3 equals the
    independent C oracle's beta (fp64 mode), and the fp16-operand form stays within the fp16
    rounding of it; imposing the computed masks reproduces mlp_backward."""
    from oracle import adjoint
    spec = synth.custom("mlpp", 403, B=1, C=1, H=5, W=7, K=9, S=3, h1=24, h2=20)
    inp = synth.make_inputs(spec)
    z = inp.zernike[0].astype(np.float64)
    ref = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)[0].reshape(9, -1)
    for prec, tol in (("fp64", 1e-12), ("fp16", 5e-3)):
        p1, p2 = adjoint.mlp_preactivations(z, inp.mlp, prec)
        beta = inp.mlp["W3"].astype(np.float64) @ np.maximum(p2, 0) + inp.mlp["b3"].astype(np.float64)[:, None]
        assert np.abs(beta - ref).max() <= tol * (1 + np.abs(ref).max()), prec
    g = np.random.default_rng(5).standard_normal((9, 5, 7))
    p1, p2 = adjoint.mlp_preactivations(z, inp.mlp, "fp16")
    np.testing.assert_array_equal(adjoint.mlp_backward(z, g, inp.mlp, masks=(p1 > 0, p2 > 0)),
                                  adjoint.mlp_backward(z, g, inp.mlp, "fp16"))


def test_anchors_backward_is_the_transpose_of_the_c_interpolation():
    """dL/dA = Wy^T dL/dz Wx is pinned against the independent C oracle of the forward
    interpolation (p2s_oracle_interp_anchors) by the dot-product identity <g, interp(A)> =
    <interp^T(g), A>, for several G (1, 2, 5, 16) and ragged H, W; plus closed forms: each pixel's
    weights sum to 1, so sum(dL/dA) = sum(dL/dz), and a constant dL/dz = 1 gives
    dL/dA[a][b] = (sum_y Wy[y][a]) (sum_x Wx[x][b])."""
    from oracle import adjoint
    rng = np.random.default_rng(8)
    for G, H, W in ((1, 7, 9), (2, 5, 13), (5, 37, 29), (16, 64, 40)):
        A = rng.standard_normal((2, 3, G, G)).astype(np.float32)
        g = rng.standard_normal((2, 3, H, W))
        z = oracle.interp_anchors(A, H, W)
        gA = adjoint.anchors_backward(g, G)
        lhs, rhs = np.sum(g * z), np.sum(gA * A.astype(np.float64))
        assert abs(lhs - rhs) <= 1e-10 * (1 + abs(lhs)), (G, lhs, rhs)
        np.testing.assert_allclose(gA.sum(axis=(2, 3)), g.sum(axis=(2, 3)), rtol=1e-12, atol=1e-9)
        ones = adjoint.anchors_backward(np.ones((1, 1, H, W)), G)[0, 0]
        wy, wx = adjoint.anchor_weights(H, G).sum(0), adjoint.anchor_weights(W, G).sum(0)
        np.testing.assert_allclose(ones, np.outer(wy, wx), rtol=1e-12)


def test_backward_color_reduces_to_shared_and_matches_finite_differences():
    """Adjoint of the wavelength-dependent colour render (oracle.adjoint.backward_color): with every
    channel's field equal it is the shared-beta adjoint (dL/dbeta = sum_c dL/dbeta_c, dL/dt and
    dL/dI equal, dL/dz = sum_c dL/dz_c); with different fields, central differences of
    oracle.render_color (an independent forward) match dL/dz_c, dL/dI and dL/dt at sampled entries."""
    from oracle import adjoint
    spec = synth.custom("bcol", 404, B=1, C=3, H=6, W=7, K=4, S=3, h1=10, h2=9, t_std=0.6)
    inp = synth.make_inputs(spec)
    img, t = inp.image[0].astype(np.float64), inp.tilt[0]
    g = np.random.default_rng(6).standard_normal((3, 6, 7))
    z = inp.zernike[0]
    zc_eq = np.stack([z] * 3)
    gb, gt, gi, gz = adjoint.backward_color(img, zc_eq, t, inp.basis, inp.mlp, g)
    beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)[0]
    _, gb_s, gt_s, gi_s = adjoint.backward(img, beta, t, inp.basis, g)
    np.testing.assert_allclose(gb.sum(0), gb_s, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(gt, gt_s, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(gi, gi_s, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(gz.sum(0), adjoint.mlp_backward(z.astype(np.float64), gb_s, inp.mlp), rtol=1e-9,
                               atol=1e-12)
    # different fields per channel: finite differences of the colour render
    zc = np.stack([z * s for s in (1.0, 0.8, 1.3)]).astype(np.float32)
    gb, gt, gi, gz = adjoint.backward_color(img, zc, t, inp.basis, inp.mlp, g)

    def loss(im, zz, tt):
        o, _ = oracle.render_color(im[None].astype(np.float32), zz[None].astype(np.float32), tt[None].astype(np.float32),
                                   inp.basis, inp.mlp)
        return np.sum(g * o[0])
    rng = np.random.default_rng(7)
    for _ in range(6):
        c, j, y, x = rng.integers(0, 3), rng.integers(0, spec.n_in), rng.integers(0, 6), rng.integers(0, 7)
        e = np.zeros_like(zc)
        e[c, j, y, x] = 1e-2
        fd = (loss(img, zc + e, t) - loss(img, zc - e, t)) / 2e-2
        assert abs(fd - gz[c, j, y, x]) < 2e-4 * (1 + abs(gz[c, j, y, x])), ("z", fd, gz[c, j, y, x])
        e = np.zeros_like(img)
        e[c, y, x] = 1e-2
        fd = (loss(img + e, zc, t) - loss(img - e, zc, t)) / 2e-2
        assert abs(fd - gi[c, y, x]) < 2e-4 * (1 + abs(gi[c, y, x])), ("I", fd, gi[c, y, x])
        e = np.zeros(t.shape, np.float64)
        e[c % 2, y, x] = 1e-3
        fd = (loss(img, zc, t + e) - loss(img, zc, t - e)) / 2e-3
        assert abs(fd - gt[c % 2, y, x]) < 1e-3 * (1 + abs(gt[c % 2, y, x])), ("t", fd, gt[c % 2, y, x])


# ---------------------------------------------------------------- hand-worked fixture
def _golden_3x3():
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_3x3.json")))
    img = np.array(g["image"], np.float32)[None, None]
    z = np.array(g["zernike"], np.float32)[None, None]
    t = np.zeros((1, 2, 3, 3), np.float32)
    t[:, 0], t[:, 1] = g["tilt_x"], g["tilt_y"]
    phi = np.array(g["phi"], np.float32)
    mlp = {k: np.array(v, np.float32) for k, v in g["mlp"].items()}
    return g, img, z, t, phi, mlp


def test_golden_hand_worked_3x3_frame():
    """tests/golden/worked_3x3.json — a whole frame (MLP with a ReLU that switches at one pixel,
    two delta basis functions, half-pixel tilt) worked by hand from PAPER.md:224-235 (Eq. 4-5),
    :280-283 and :172; the file carries the derivation. The paper prints no numeric example
    (SURVEY.md:218), so the expected numbers are the hand's, not the oracle's: a correlation
    instead of a convolution, beta taken at the source pixel, a forward warp, swapped tilt planes
    or a wrong clamp each change them."""
    g, img, z, t, phi, mlp = _golden_3x3()
    out, J = oracle.render(img, z, t, phi, mlp, want_blur=True)
    b = oracle.beta(img, z, phi, mlp)
    np.testing.assert_allclose(b[0, :, 0, 0], g["beta_at_0_0"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(b[0, :, 1, 1], g["beta_at_1_1"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(J[0, 0], np.array(g["J"]), rtol=0, atol=1e-6)      # inputs are fp32
    np.testing.assert_allclose(out[0, 0], np.array(g["out"]), rtol=0, atol=1e-6)
    # swapping the tilt planes (a vertical half-pixel shift) must NOT give the same frame
    out_sw, _ = oracle.render(img, z, t[:, ::-1].copy(), phi, mlp, want_blur=True)
    assert np.abs(out_sw[0, 0] - np.array(g["out"])).max() > 0.05
