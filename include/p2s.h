/* p2s.h — C ABI of the B200-native Phase-to-Space (P2S) turbulence renderer.
 *
 * One frame = three steps of Mao, Chimitt & Chan, "Accelerating Atmospheric Turbulence
 * Simulation via Learned Phase-to-Space Transform" (ICCV 2021; /root/reference/PAPER.md):
 *   a1  P2S network: per pixel, "three fully connected layers" map the high-order Zernike
 *       coefficients to the PSF-basis coefficients beta (Sec. 3.3);
 *   a2  Eq. (5): y_n = sum_m beta_{m,n} phi_m^T x — M spatially invariant convolutions
 *       weighted at the output pixel (Sec. 3.1);
 *   a3  tilt: "locally shifting the image according to its tilt" after the blur
 *       (PAPER.md:172), the first two Zernike coefficients "displace the pixels".
 * Readings of the points the paper leaves open (true convolution, replicate borders,
 * backward bilinear warp, ReLU hidden layers, no output clamp, ...) are DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - Return a p2s_status; no C++ exception crosses the ABI. Argument/shape errors are
 *    reported synchronously before any work is queued.
 *  - "DEVICE" pointers are CUDA device pointers on the current device; "HOST" pointers are
 *    ordinary host memory. All tensors are dense, row-major, fp32, 16-byte aligned (DEVICE).
 *  - Work is queued on `stream` (NULL = legacy default stream) and is asynchronous: DEVICE
 *    inputs must stay valid and unmodified, and outputs must not be read, until the
 *    stream has reached the work. Asynchronous faults surface at the caller's next sync.
 *  - A handle owns device copies of the basis/weights plus a workspace; it serves one
 *    stream at a time (use one handle per concurrently rendering stream).
 *  - Envelope (else P2S_ERR_UNSUPPORTED): S odd, 1 <= S <= 65; 1 <= K <= 128;
 *    1 <= n_in <= 64; 1 <= h1, h2 <= 256; C in {1,2,3}; B, H, W >= 1; S*S >= 1;
 *    device = sm_100 (B200).
 */
#ifndef P2S_H
#define P2S_H

#if defined(__GNUC__)
#define P2S_API __attribute__((visibility("default")))
#else
#define P2S_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  P2S_OK = 0,
  P2S_ERR_INVALID_ARG = 1, /* null pointer, inconsistent dims, aliasing output */
  P2S_ERR_UNSUPPORTED = 2, /* outside the envelope above, or not an sm_100 device */
  P2S_ERR_CUDA = 3,        /* a CUDA runtime/launch error (see p2s_last_cuda_error) */
  P2S_ERR_OOM = 4          /* device allocation failed */
} p2s_status;

typedef struct CUstream_st* p2s_stream_t; /* == cudaStream_t */
typedef struct CUevent_st* p2s_event_t;   /* == cudaEvent_t  */
typedef struct p2s_handle p2s_handle;     /* opaque */

/* PSF basis phi_k, k = 0..K-1 (the paper's M basis functions).
 * HOST pointer to [K][S][S] fp32 row-major; taps[k][i][j] is the tap at offset
 * (dy, dx) = (i - r, j - r), r = (S-1)/2, applied as a TRUE convolution (A2/A3). */
typedef struct {
  int K, S;
  const float* taps;
} p2s_basis;

/* P2S network: beta = W3 relu(W2 relu(W1 z + b1) + b2) + b3.
 * HOST pointers, torch.nn.Linear layout: W1 [h1][n_in], W2 [h2][h1], W3 [n_out][h2] row-major,
 * b* [out]. n_out must equal the basis K. */
typedef struct {
  int n_in, h1, h2, n_out;
  const float *W1, *b1, *W2, *b2, *W3, *b3;
} p2s_mlp;

/* Source image x of Eq. (3): DEVICE [B][C][H][W] fp32 (values in [0,1]
 * for the stated tolerance; any finite values are accepted). Channels share beta and tilt
 * (PAPER.md:320). */
typedef struct {
  const float* data;
  int B, C, H, W;
} p2s_image;

/* Deep-copies and repacks `basis` and `mlp_weights` (the caller may free them on return):
 * taps are flipped/regrouped into the tensor-core operand layout and converted to fp16,
 * weights to fp16, biases and tap sums kept in fp32. Allocates device memory on the
 * current device. On success *out_handle owns everything; release with p2s_destroy. */
P2S_API p2s_status p2s_init(const p2s_basis* basis, const p2s_mlp* mlp_weights, p2s_handle** out_handle);

/* Renders B frames: out = warp_t( J ), J_c = sum_k beta_k (I_c * phi_k), beta = P2S(z).
 *   zernike_field DEVICE [B][n_in][H][W] fp32: per-pixel high-order Zernike coefficients
 *                 (Noll Z4..Z36 for n_in = 33; "last K-2 coefficients").
 *   tilt_field    DEVICE [B][2][H][W] fp32, in pixels; channel 0 = x (columns, alpha_2),
 *                 channel 1 = y (rows, alpha_3). May be NULL (= zero tilt).
 *                 out(y,x) = bilinear J at (y - t1, x - t0), clamp-to-edge.
 *   out           DEVICE [B][C][H][W] fp32; must not overlap any input.
 * No host synchronisation and no allocation, except the first use or growth of the
 * handle's workspace (B*C*H*W fp32), which synchronises the device; p2s_reserve avoids it. */
P2S_API p2s_status p2s_render(p2s_handle* h, p2s_image image, const float* zernike_field,
                      const float* tilt_field, float* out, p2s_stream_t stream);

/* Same computation with HOST buffers (same shapes as p2s_render): copies the inputs to the
 * handle's device staging buffers, renders, copies `out` back, and synchronises `stream`
 * before returning. Host buffers should be pinned for full copy bandwidth. */
P2S_API p2s_status p2s_render_host(p2s_handle* h, const float* image_host, int B, int C, int H, int W,
                           const float* zernike_host, const float* tilt_host, float* out_host,
                           p2s_stream_t stream);

/* Anchor-grid input (Sec. 3.4: "partition the image
 * into a user-defined grid of anchor points ... interpolate the Zernike coefficients using
 * bilinear interpolation"). Instead of a dense [B][33][H][W] field the caller passes anchors
 * DEVICE [B][n_in][G][G] fp32 (G >= 1; G = 1 is a constant field); the fused kernel
 * interpolates them per pixel while staging the MLP input (phase-domain interpolation, then the
 * P2S network per pixel: PAPER.md:293-299). Registration (reading N1): pixel (y, x)
 * has centre (y + 0.5, x + 0.5); anchor (i, j) sits at (i H/(G-1), j W/(G-1)), i.e. the grid
 * spans the image corner to corner. Otherwise identical to p2s_render (tilt, out, stream,
 * ownership, errors; G outside [1, 4096] or NULL anchors -> P2S_ERR_INVALID_ARG). */
P2S_API p2s_status p2s_render_anchors(p2s_handle* h, p2s_image image, const float* anchors, int G,
                                      const float* tilt_field, float* out, p2s_stream_t stream);
/* p2s_render_anchors with HOST buffers (image, anchors [B][n_in][G][G], tilt, out), copies
 * inside, synchronous (the e2e path of the anchor mode). */
P2S_API p2s_status p2s_render_anchors_host(p2s_handle* h, const float* image_host, int B, int C, int H,
                                           int W, const float* anchors_host, int G,
                                           const float* tilt_host, float* out_host, p2s_stream_t stream);

/* Sequence mode: F degraded frames of ONE image, the way the paper's
 * training data is made ("5000 simulated sequences, where each sequence contains
 * 50 degraded frames" of one ground-truth image), each with its own Zernike field and tilt.
 * out[f] = p2s_render(image, zernike[f], tilt[f]) for every f. The K basis convolutions of the
 * image (83-93 % of the work) are computed once per tile and stay in tensor memory while the
 * P2S network and the Eq. 5 reduction run for every frame.
 * image DEVICE [1][C][H][W]; zernike_field DEVICE [F][n_in][H][W]; tilt_field DEVICE [F][2][H][W]
 * or NULL; out DEVICE [F][C][H][W]. Errors as p2s_render; image.B != 1 or F outside [1, 65535]
 * -> P2S_ERR_INVALID_ARG. */
P2S_API p2s_status p2s_render_sequence(p2s_handle* h, p2s_image image, const float* zernike_field,
                                       const float* tilt_field, int F, float* out, p2s_stream_t stream);

/* Wavelength-dependent colour ("3 PSFs with wavelengths
 * 450nm, 540nm, and 570nm ... requires 3x computation"): every channel c of frame b has its own
 * Zernike field, hence its own beta (PSF field):
 *   out[b][c] = warp(J_c, tilt[b]),  J_c(p) = sum_k beta_k(z[b][c](p)) (I[b][c] * phi_k)(p)
 * zernike_field: DEVICE [B][C][n_in][H][W] fp32 (channel-major per frame); image, tilt and out as
 * p2s_render. The K convolutions of each tile are computed once and serve the C MLP passes
 * (one fused launch; the channel passes reuse the sequence-mode schedule). With every channel's
 * field equal this is p2s_render. Errors as p2s_render. */
P2S_API p2s_status p2s_render_color(p2s_handle* h, p2s_image image, const float* zernike_field,
                                    const float* tilt_field, float* out, p2s_stream_t stream);

/* Adjoint of steps a2-a3 ("differentiable module"): for the
 * frames p2s_render would produce and an upstream gradient grad_out = dL/dout (DEVICE
 * [B][C][H][W] fp32), writes
 *   grad_beta (DEVICE [B][K][H][W] or NULL) = dL/dbeta_k(p) = sum_c dL/dJ_c(p) C_kc(p)
 *   grad_tilt (DEVICE [B][2][H][W] or NULL) = dL/dt(p) through the bilinear warp (0 where the
 *     coordinate clamp is active)
 *   grad_image (DEVICE [B][C][H][W] or NULL) = dL/dI_c(q) = sum over the taps that read q (after
 *     the replicate clamp) of phi_k[i][j] beta_k(p) dL/dJ_c(p): the transpose of Eq. 5's
 *     beta-weighted convolution ("scatter order"), on the tensor cores with U = beta dL/dJ
 *     rounded to fp16 after scaling each (frame, channel) plane by a power of two (any finite
 *     grad_out range; the sums are scaled back)
 * where dL/dJ scatters grad_out through the warp's bilinear weights (float atomics: the
 * summation order, hence the last bits, vary run to run; grad_image's border pixels likewise).
 * grad_beta recomputes the K convolutions on the tensor cores; grad_tilt also recomputes J (one
 * forward); grad_image recomputes beta (one MLP pass, in the forward's fused kernel) and needs
 * workspace for dL/dJ [B][C][H][W] fp32 and U [B][C][K][H][ceil8(W)] fp16 (grown on first use:
 * synchronising, like p2s_render's; p2s_reserve_ex pre-sizes them). Errors as p2s_render; all
 * three outputs NULL, or an output overlapping an input or another output -> P2S_ERR_INVALID_ARG. */
P2S_API p2s_status p2s_backward(p2s_handle* h, p2s_image image, const float* zernike_field,
                                const float* tilt_field, const float* grad_out, float* grad_beta,
                                float* grad_tilt, float* grad_image, p2s_stream_t stream);

/* dL/dz through the P2S MLP (the adjoint of step a1; "three fully connected
 * layers", reading A11: ReLU after layers 1-2, linear output; "differentiable
 * module"). For the Zernike field zernike_field (DEVICE [B][n_in][H][W] fp32, the p2s_render
 * input) and grad_beta = dL/dbeta (DEVICE [B][K][H][W] fp32, e.g. p2s_backward's grad_beta), writes
 *   grad_zernike (DEVICE [B][n_in][H][W] fp32) = W1^T ((W2^T ((W3^T grad_beta) [pre2 > 0])) [pre1 > 0])
 * per pixel, pre1 = W1 z + b1, pre2 = W2 ReLU(pre1) + b2 (the forward masks are recomputed).
 * Tensor cores with fp16 operands and fp32 accumulation; grad_beta is scaled per pixel by a power
 * of two before rounding (any finite range); the masks are decided on the fp16-operand fp32
 * accumulators (reading N5), so a pre-activation within rounding of 0 may take
 * either side. Asynchronous on `stream`; no allocation. Errors: NULL pointers, B/H/W < 1 or
 * grad_zernike overlapping an input -> P2S_ERR_INVALID_ARG; frames whose channel planes exceed
 * 2^31 elements -> P2S_ERR_UNSUPPORTED; launch failure -> P2S_ERR_CUDA. MLPs whose weights do not
 * all fit one SM next to the activation tile (e.g. 33-256-256-100) run a variant that streams
 * the weights from L2, two CTAs per SM; every MLP p2s_init accepts is supported
 * (p2s_info.mlp_backward = 1). */
P2S_API p2s_status p2s_mlp_backward(p2s_handle* h, const float* zernike_field, const float* grad_beta, int B,
                                    int H, int W, float* grad_zernike, p2s_stream_t stream);

/* Adjoint of p2s_render_color (SURVEY §8(f) row 5 with NEXT-4): channel c
 * of frame b is a one-channel render with its own field z[b][c], so for grad_out = dL/dout
 * (DEVICE [B][C][H][W]) it writes
 *   grad_beta    (DEVICE [B][C][K][H][W] or NULL)     dL/dbeta_c of each channel's own beta
 *   grad_tilt    (DEVICE [B][2][H][W] or NULL)        summed over the channels
 *   grad_image   (DEVICE [B][C][H][W] or NULL)
 *   grad_zernike (DEVICE [B][C][n_in][H][W] or NULL)  dL/dz_c through the MLP (p2s_mlp_backward)
 * as ONE p2s_backward over the B*C one-channel frames the colour layouts already are (tilt
 * replicated per channel) and one p2s_mlp_backward (their precision notes apply). zernike_field
 * as p2s_render_color. Workspace (replicated tilt and per-channel dL/dt [B*C][2][H][W]; dL/dbeta
 * [B*C][K][H][W] when only dL/dz is wanted) grows on first use (synchronising). Errors as
 * p2s_backward; all four outputs NULL -> P2S_ERR_INVALID_ARG. */
P2S_API p2s_status p2s_backward_color(p2s_handle* h, p2s_image image, const float* zernike_field,
                                      const float* tilt_field, const float* grad_out, float* grad_beta,
                                      float* grad_tilt, float* grad_image, float* grad_zernike,
                                      p2s_stream_t stream);

/* The anchor-grid interpolation ("anchor points ... interpolated"; registration
 * DESIGN.md reading N1 — pixel centre (t + 0.5), anchors at a n / (G - 1)) as a standalone op and
 * its adjoint, so the anchor pipeline is differentiable end to end:
 *   p2s_interp_anchors:  anchors (DEVICE [B][n_in][G][G] fp32) -> zernike_field (DEVICE
 *     [B][n_in][H][W] fp32), z = Wy A Wx^T per frame and mode, the fp32 arithmetic of
 *     p2s_render_anchors' staging (p2s_render on this field equals p2s_render_anchors);
 *   p2s_anchors_backward: grad_zernike (DEVICE [B][n_in][H][W]) -> grad_anchors (DEVICE
 *     [B][n_in][G][G]) = Wy^T grad_zernike Wx (deterministic: a fixed reduction order).
 * Handle-free; asynchronous on `stream`; NULL pointers, B/n_in/H/W < 1, G outside [1, 4096] or
 * an output overlapping the input -> P2S_ERR_INVALID_ARG; launch failure -> P2S_ERR_CUDA. */
P2S_API p2s_status p2s_interp_anchors(const float* anchors, int B, int n_in, int G, int H, int W,
                                      float* zernike_field, p2s_stream_t stream);
P2S_API p2s_status p2s_anchors_backward(const float* grad_zernike, int B, int n_in, int G, int H, int W,
                                        float* grad_anchors, p2s_stream_t stream);

/* ---- correlated anchor sampling (Sec. 3.4: anchor
 * coefficient sets "drawn from the correlation matrix", which "can be pre-computed") ----
 * Stand-in covariance (reading N3; the paper's Takato-formula parameters are absent):
 * separable over anchor row a, anchor column b and mode j:
 *   Cov[A_j(a,b), A_j'(a',b')] = R[j][j'] s(a-a') s(b-b'), s(d) = exp(-d^2/(2 l^2)) + 1e-6 [d = 0]
 * with l = corr_len in anchor spacings (0: independent anchors) and R = mode_cov (HOST fp64
 * [n_in][n_in], symmetric positive definite; NULL: 0.25 I). p2s_sampler_init factors both
 * (Cholesky, fp64, once); p2s_sample_anchors writes F frames A_f = (L_R (x) L_s (x) L_s) z_f to
 * anchors (DEVICE [F][n_in][G][G] fp32, the layout p2s_render_anchors reads), z_f ~ N(0, I) from
 * Philox4x32-10 (key = seed, counter = (frame0 + f, a G + b, j, 0)) + Box-Muller: every frame is
 * reproducible on its own. G in [1, 64], n_in in [1, 64]; a non-SPD mode_cov, a bad size or NULL
 * pointers -> P2S_ERR_INVALID_ARG. Asynchronous on `stream`. */
typedef struct p2s_sampler p2s_sampler;
P2S_API p2s_status p2s_sampler_init(int G, int n_in, double corr_len, const double* mode_cov,
                                    p2s_sampler** out_sampler);
/* Dense pre-computed correlation ("This grid corresponds to a correlation matrix of
 * size 64^2 x 64^2 = 4096 x 4096 which can be pre-computed ... 4096 sets of Zernike coefficients
 * are drawn from the correlation matrix"; the Takato-formula entries of P:295 need parameters the
 * paper does not give, reading N6):
 *   Cov[A_j(p), A_j'(p')] = R[j][j'] C[p][p'],  p = a G + b (anchor row a, column b),
 * spatial_cov = C: HOST fp64 [G^2][G^2] row-major, symmetric positive definite, factored once here
 * (fp64 Cholesky on the host, threaded; ~1 s at G = 64); or, with is_factor != 0, its lower
 * Cholesky factor L (the upper triangle is ignored, the diagonal must be > 0). mode_cov as
 * p2s_sampler_init. The sampler owns device copies of L (fp16 hi/lo tiles, ~33 MB at G = 64) and a
 * workspace; p2s_sample_anchors then draws A_f = (L_R (x) L) z_f with the same Philox normals z_f
 * as the separable sampler (so C = s (x) s reproduces it up to rounding), the product L Y as a
 * tcgen05 GEMM over L's lower triangle with fp16 hi/lo operand splits (lo parts scaled by 2^11, L
 * by 2^14) and fp32 accumulation:
 * |error| <= ~2^-20 x sum_q |L[p][q]| |Y[q]| per anchor. Errors: NULL
 * spatial_cov / out, G outside [1, 64], n_in outside [1, 64], a non-symmetric or non-SPD matrix
 * -> P2S_ERR_INVALID_ARG; not an sm_100 device -> P2S_ERR_UNSUPPORTED; allocation -> P2S_ERR_OOM. */
P2S_API p2s_status p2s_sampler_init_dense(int G, int n_in, const double* spatial_cov, int is_factor,
                                          const double* mode_cov, p2s_sampler** out_sampler);
P2S_API p2s_status p2s_sample_anchors(p2s_sampler* s, unsigned long long seed, int frame0, int F,
                                      float* anchors, p2s_stream_t stream);
P2S_API void p2s_sampler_destroy(p2s_sampler* s);

/* Pre-sizes the render workspace (J, B*C*H*W fp32) for frames up to B x C x H x W, so that later
 * p2s_render / p2s_render_sequence / p2s_render_color calls of that size neither allocate nor
 * synchronise (and can be captured in a CUDA graph). Synchronises the device when it grows the
 * workspace. Errors: NULL handle or a size < 1 -> P2S_ERR_INVALID_ARG; P2S_ERR_CUDA / OOM. */
P2S_API p2s_status p2s_reserve(p2s_handle* h, int B, int C, int H, int W);

/* p2s_reserve with a choice of workspaces (bitwise OR of P2S_RESERVE_*), for frames up to
 * B x C x H x W: RENDER = the render workspace (as p2s_reserve); HOST = also the device staging
 * of p2s_render_host / p2s_render_anchors_host (image, out, Zernike field, tilt) and its input
 * stream; ADJOINT = also p2s_backward's dL/dJ buffer (enough for grad_beta / grad_tilt);
 * ADJOINT_IMAGE = also its grad_image workspaces (U = beta dL/dJ, fp16 [B][C][K][H][ceil8(W)],
 * and the per-(frame, channel) range exponents). After it, calls of at most that size allocate
 * nothing and do not synchronise. Errors: as p2s_reserve; unknown bits -> P2S_ERR_INVALID_ARG. */
#define P2S_RESERVE_RENDER 1u
#define P2S_RESERVE_HOST 2u
#define P2S_RESERVE_ADJOINT 4u
#define P2S_RESERVE_ADJOINT_IMAGE 8u
P2S_API p2s_status p2s_reserve_ex(p2s_handle* h, int B, int C, int H, int W, unsigned what);

/* When both events are non-NULL, every later p2s_render records ev_begin right before the
 * fused MLP+convolution kernel and ev_end right after it on the render stream (so its
 * duration can be timed alone); pass NULLs to stop. Events stay owned by the caller. */
P2S_API p2s_status p2s_set_profile_events(p2s_handle* h, p2s_event_t ev_begin, p2s_event_t ev_end);

/* Static facts about the handle's execution plan (for reports/tests). */
typedef struct {
  int K, S, n_in, h1, h2;
  int n_pad, h1_pad, h2_pad, in_pad; /* tensor-core padded dims */
  int conv_steps;                    /* 16-tap K-slices per channel (sum of taps padded) */
  int smem_bytes;                    /* dynamic shared memory of the fused kernel */
  int kernels_per_render;            /* launches queued by one p2s_render */
  int stage_bytes, nring;            /* B-operand ring: bytes per stage, stages */
  int mlp_backward;                  /* 1: p2s_mlp_backward supports this MLP (all p2s_init accepts) */
  int c1_plan;                       /* 1: one-channel calls run on a one-channel plan (E buffers and
                                        TMEM for C = 1; one op per MLP layer) */
  int c1_smem_bytes, c1_nring, c1_stage_bytes; /* that plan's shared memory and ring (0 if none) */
  int seq_plan;                      /* 1: p2s_render_sequence (C > 1) runs on a half-E plan of its own
                                        (two half-size E buffers, a larger operand ring) */
  int seq_nring, seq_stage_bytes;    /* that plan's ring (0 if none) */
} p2s_info;
P2S_API p2s_status p2s_get_info(const p2s_handle* h, p2s_info* info);

/* Releases every resource of the handle (synchronises the device). NULL is a no-op. */
P2S_API void p2s_destroy(p2s_handle* h);

/* Static string for a status code. */
P2S_API const char* p2s_status_string(p2s_status s);

/* Message of the last CUDA error seen by this library on this thread ("" if none). */
P2S_API const char* p2s_last_cuda_error(void);

/* ---- test/debug taps (same stream semantics as p2s_render) ----
 * p2s_debug_beta: step a1 only; beta_out DEVICE [B][K][H][W] fp32.
 * p2s_debug_blur: steps a1+a2 only (no warp); J_out DEVICE [B][C][H][W] fp32. */
P2S_API p2s_status p2s_debug_beta(p2s_handle* h, const float* zernike_field, int B, int H, int W,
                          float* beta_out, p2s_stream_t stream);
/* p2s_debug_blur_anchors: steps a1+a2 from an anchor grid (as p2s_render_anchors), no warp. */
P2S_API p2s_status p2s_debug_blur_anchors(p2s_handle* h, p2s_image image, const float* anchors, int G,
                                          float* J_out, p2s_stream_t stream);
P2S_API p2s_status p2s_debug_blur(p2s_handle* h, p2s_image image, const float* zernike_field,
                          float* J_out, p2s_stream_t stream);
/* p2s_debug_profile_buffer: in a library built with -DP2S_PROFILE, later launches write per-CTA
 * role timers (clock64 cycles; layout documented in tools/role_profile.py) to
 * device_counters [grid][4][20] u64; NULL disables. Other builds return P2S_ERR_UNSUPPORTED. */
P2S_API p2s_status p2s_debug_profile_buffer(p2s_handle* h, void* device_counters);

#ifdef __cplusplus
}
#endif
#endif /* P2S_H */
