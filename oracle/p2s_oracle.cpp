// p2s_oracle.cpp — plain, slow, obviously-correct CPU oracle for the P2S hot path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load this library. The product path
// (paper_2107_11627_b200, the C-ABI in include/p2s.h) never links or calls it, and the
// two share no code: no headers, helpers, tables or constants.
//
// What it computes (fp32 inputs, fp64 arithmetic, results returned in fp64), for every
// frame b and pixel (y, x); cY(v) = min(max(v,0),H-1), cX likewise; r = (S-1)/2:
//
//  step a1 — P2S network, "three fully connected layers" mapping the high-order Zernike
//    coefficients of a pixel to its PSF-basis coefficients (Sec. 3.3):
//      a1 = ReLU(W1 z + b1), a2 = ReLU(W2 a1 + b2), beta = W3 a2 + b3   (no output act.)
//    (readings A9/A11/A14 of DESIGN.md: 33 inputs Z4..Z36, ReLU hidden, linear output)
//
//  step a2 — Eq. (5): y_n = sum_m beta_{m,n} phi_m^T x, i.e. M
//    spatially invariant convolutions combined per output pixel ("gather" order, A1):
//      C_k(y,x) = sum_{i,j} phi_k[i][j] * I[cY(y-(i-r))][cX(x-(j-r))]   (true conv, A2-A4)
//      J(y,x)   = sum_k beta_k(y,x) * C_k(y,x)
//    Colour channels share beta (A13).
//
//  step a3 — tilt: "locally shifting the image according to its tilt" after the blur
//    (PAPER.md:172), "uses the first two Zernike coefficients to displace the pixels"
//    (PAPER.md:280). Backward bilinear warp, clamp-to-edge (A5-A8):
//      sy = y - t1(y,x), sx = x - t0(y,x) (clamped to [-1,H] / [-1,W], which changes
//      nothing but keeps floor() in int range); y0 = floor(sy), fy = sy - y0, ...
//      out = (1-fy)(1-fx) J[cY(y0)][cX(x0)] + (1-fy) fx J[cY(y0)][cX(x0+1)]
//          + fy (1-fx) J[cY(y0+1)][cX(x0)] + fy fx J[cY(y0+1)][cX(x0+1)]
//    No output clamp (A12).
//
//  anchor grid (Sec. 3.4 "partition the image into a
//    user-defined grid of anchor points ... interpolate the Zernike coefficients using
//    bilinear interpolation"): a G x G grid of coefficient vectors, registered to the image
//    corners with half-pixel alignment (reading N1): pixel (y, x) has continuous
//    centre (y + 0.5, x + 0.5) in [0, H] x [0, W]; anchor (i, j) sits at (i H/(G-1), j W/(G-1)).
//      u = (y + 0.5)(G-1)/H, i0 = min(floor(u), G-2), fy = u - i0   (v, j0, fx likewise)
//      z_k(y,x) = (1-fy)(1-fx) A_k[i0][j0] + (1-fy) fx A_k[i0][j0+1]
//               + fy (1-fx) A_k[i0+1][j0] + fy fx A_k[i0+1][j0+1]      (each mode k separately)
//    G = 1: constant field. The dense field then feeds step a1 exactly as a given field does.
//
//  adjoint of step a2 ("differentiable module"), for a given
//    beta [K] per pixel and upstream dL/dJ = gJ [C] per pixel (fp64 inputs):
//      dL/dbeta_k(y,x) = sum_c gJ_c(y,x) C_kc(y,x)                     (C_kc as in step a2)
//      dL/dI_c(q)      = sum over pixels p and taps (i,j) with (cY(p_y-(i-r)), cX(p_x-(j-r))) = q
//                        of phi_k[i][j] beta_k(p) gJ_c(p)               (the transpose of Eq. 5:
//                        every term of J_c(p) sends its weight back to the pixel it read)
//
// Parity pins for every function live in tests/test_oracle_pins.py (closed forms,
// invariants, library routines: torch nn.Linear, scipy.ndimage.convolve,
// torch grid_sample, FFT convolution).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <algorithm>
#include <atomic>

namespace {

struct Problem {
  int B, C, H, W;
  int n_in, h1, h2, K, S;
  const float *image, *zernike, *tilt, *taps;
  const float *W1, *b1, *W2, *b2, *W3, *b3;
};

inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Step a1 at one pixel: beta[K].
void mlp_pixel(const Problem& p, int b, int y, int x, double* beta) {
  const size_t HW = (size_t)p.H * p.W, pix = (size_t)y * p.W + x;
  std::vector<double> z(p.n_in), a1(p.h1), a2(p.h2);
  for (int j = 0; j < p.n_in; ++j) z[j] = p.zernike[((size_t)b * p.n_in + j) * HW + pix];
  for (int o = 0; o < p.h1; ++o) {
    double s = p.b1[o];
    for (int i = 0; i < p.n_in; ++i) s += (double)p.W1[(size_t)o * p.n_in + i] * z[i];
    a1[o] = s > 0.0 ? s : 0.0;
  }
  for (int o = 0; o < p.h2; ++o) {
    double s = p.b2[o];
    for (int i = 0; i < p.h1; ++i) s += (double)p.W2[(size_t)o * p.h1 + i] * a1[i];
    a2[o] = s > 0.0 ? s : 0.0;
  }
  for (int o = 0; o < p.K; ++o) {
    double s = p.b3[o];
    for (int i = 0; i < p.h2; ++i) s += (double)p.W3[(size_t)o * p.h2 + i] * a2[i];
    beta[o] = s;
  }
}

// Step a2 at one pixel, all channels: J[c] = sum_k beta_k * (I_c * phi_k)(y,x) (Eq. 5).
void blur_pixel(const Problem& p, int b, int y, int x, const double* beta, double* J) {
  const int S = p.S, r = (S - 1) / 2;
  const size_t HW = (size_t)p.H * p.W;
  std::vector<double> patch((size_t)S * S);
  for (int c = 0; c < p.C; ++c) {
    const float* img = p.image + ((size_t)b * p.C + c) * HW;
    // patch[i][j] = I[cY(y-(i-r))][cX(x-(j-r))]  (true convolution, replicate edges)
    for (int i = 0; i < S; ++i) {
      const int yy = clampi(y - (i - r), 0, p.H - 1);
      for (int j = 0; j < S; ++j) {
        const int xx = clampi(x - (j - r), 0, p.W - 1);
        patch[(size_t)i * S + j] = img[(size_t)yy * p.W + xx];
      }
    }
    double acc = 0.0;
    for (int k = 0; k < p.K; ++k) {
      const float* phi = p.taps + (size_t)k * S * S;
      double ck = 0.0;
      for (int t = 0; t < S * S; ++t) ck += (double)phi[t] * patch[t];
      acc += beta[k] * ck;
    }
    J[c] = acc;
  }
}

// Step a3 at one pixel given a J lookup: out = bilinear J at (y - t1, x - t0), clamp-to-edge.
template <class JFn>
void warp_pixel(const Problem& p, int b, int y, int x, JFn Jat, double* out) {
  const size_t HW = (size_t)p.H * p.W, pix = (size_t)y * p.W + x;
  double tx = 0.0, ty = 0.0;
  if (p.tilt) {
    tx = p.tilt[((size_t)b * 2 + 0) * HW + pix];
    ty = p.tilt[((size_t)b * 2 + 1) * HW + pix];
  }
  double sy = (double)y - ty, sx = (double)x - tx;
  sy = std::min(std::max(sy, -1.0), (double)p.H);
  sx = std::min(std::max(sx, -1.0), (double)p.W);
  const double fy0 = std::floor(sy), fx0 = std::floor(sx);
  const double fy = sy - fy0, fx = sx - fx0;
  const int y0 = (int)fy0, x0 = (int)fx0;
  const int ya = clampi(y0, 0, p.H - 1), yb = clampi(y0 + 1, 0, p.H - 1);
  const int xa = clampi(x0, 0, p.W - 1), xb = clampi(x0 + 1, 0, p.W - 1);
  for (int c = 0; c < p.C; ++c) {
    out[c] = (1 - fy) * (1 - fx) * Jat(c, ya, xa) + (1 - fy) * fx * Jat(c, ya, xb) +
             fy * (1 - fx) * Jat(c, yb, xa) + fy * fx * Jat(c, yb, xb);
  }
}

template <class F>
void parallel_rows(int H, int nthreads, F f) {
  if (nthreads <= 1) { for (int y = 0; y < H; ++y) f(y); return; }
  std::vector<std::thread> th;
  std::atomic_int next{0};
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&]() { for (int y; (y = next.fetch_add(1)) < H;) f(y); });
  for (auto& t : th) t.join();
}

Problem make_problem(const float* image, int B, int C, int H, int W, const float* zernike,
                     int n_in, const float* tilt, const float* taps, int K, int S, int h1,
                     int h2, const float* W1, const float* b1, const float* W2,
                     const float* b2, const float* W3, const float* b3) {
  Problem p{B, C, H, W, n_in, h1, h2, K, S, image, zernike, tilt, taps, W1, b1, W2, b2, W3, b3};
  return p;
}

bool bad(const Problem& p) {
  return p.B < 1 || p.C < 1 || p.H < 1 || p.W < 1 || p.n_in < 1 || p.h1 < 1 || p.h2 < 1 ||
         p.K < 1 || p.S < 1 || (p.S % 2) == 0 || !p.image || !p.zernike || !p.taps || !p.W1 ||
         !p.b1 || !p.W2 || !p.b2 || !p.W3 || !p.b3;
}

}  // namespace

extern "C" {

#define ORACLE_ARGS                                                                        \
  const float *image, int B, int C, int H, int W, const float *zernike, int n_in,          \
      const float *tilt, const float *taps, int K, int S, int h1, int h2, const float *W1, \
      const float *b1, const float *W2, const float *b2, const float *W3, const float *b3
#define ORACLE_PASS image, B, C, H, W, zernike, n_in, tilt, taps, K, S, h1, h2, W1, b1, W2, b2, W3, b3

// beta_out [B][K][H][W] fp64 for rows [y_begin, y_end) of every frame. Returns 0 / -1.
int p2s_oracle_beta(ORACLE_ARGS, int y_begin, int y_end, double* beta_out, int nthreads) {
  Problem p = make_problem(ORACLE_PASS);
  if (bad(p) || !beta_out) return -1;
  y_begin = std::max(0, y_begin); y_end = std::min(H, y_end);
  const size_t HW = (size_t)H * W;
  for (int b = 0; b < B; ++b)
    parallel_rows(y_end - y_begin, nthreads, [&](int yi) {
      const int y = y_begin + yi;
      std::vector<double> beta(K);
      for (int x = 0; x < W; ++x) {
        mlp_pixel(p, b, y, x, beta.data());
        for (int k = 0; k < K; ++k) beta_out[((size_t)b * K + k) * HW + (size_t)y * W + x] = beta[k];
      }
    });
  return 0;
}

// Full render. J_out (optional) [B][C][H][W] fp64 = blur before warp; out [B][C][H][W] fp64.
// Rows [y_begin, y_end) of `out` are produced (J is computed on every row the warp reads).
int p2s_oracle_render(ORACLE_ARGS, int y_begin, int y_end, double* J_out, double* out,
                      int nthreads) {
  Problem p = make_problem(ORACLE_PASS);
  if (bad(p)) return -1;
  y_begin = std::max(0, y_begin); y_end = std::min(H, y_end);
  if (y_end <= y_begin) return 0;
  const size_t HW = (size_t)H * W;
  std::vector<double> J((size_t)C * HW, 0.0);
  std::vector<char> need(H, 0);
  for (int b = 0; b < B; ++b) {
    // rows of J the warp of rows [y_begin, y_end) can touch
    std::fill(need.begin(), need.end(), 0);
    for (int y = y_begin; y < y_end; ++y)
      for (int x = 0; x < W; ++x) {
        double ty = p.tilt ? p.tilt[((size_t)b * 2 + 1) * HW + (size_t)y * W + x] : 0.0;
        double sy = std::min(std::max((double)y - ty, -1.0), (double)H);
        int y0 = (int)std::floor(sy);
        need[clampi(y0, 0, H - 1)] = 1;
        need[clampi(y0 + 1, 0, H - 1)] = 1;
      }
    parallel_rows(H, nthreads, [&](int y) {
      if (!need[y] && !J_out) return;
      std::vector<double> beta(K), jc(C);
      for (int x = 0; x < W; ++x) {
        mlp_pixel(p, b, y, x, beta.data());
        blur_pixel(p, b, y, x, beta.data(), jc.data());
        for (int c = 0; c < C; ++c) J[(size_t)c * HW + (size_t)y * W + x] = jc[c];
      }
    });
    if (J_out) std::memcpy(J_out + (size_t)b * C * HW, J.data(), sizeof(double) * C * HW);
    if (out) {
      auto Jat = [&](int c, int yy, int xx) { return J[(size_t)c * HW + (size_t)yy * W + xx]; };
      parallel_rows(y_end - y_begin, nthreads, [&](int yi) {
        const int y = y_begin + yi;
        std::vector<double> o(C);
        for (int x = 0; x < W; ++x) {
          warp_pixel(p, b, y, x, Jat, o.data());
          for (int c = 0; c < C; ++c) out[((size_t)b * C + c) * HW + (size_t)y * W + x] = o[c];
        }
      });
    }
  }
  return 0;
}

// Sampled outputs computed one by one: for each (b, y, x) in `bxy` (n triples), J at that
// pixel (J_out[n][C], optional) and the warped output (out[n][C], optional). Each output
// evaluates the MLP + Eq. (5) at its four bilinear neighbours directly.
int p2s_oracle_pixels(ORACLE_ARGS, const int* bxy, int n, double* J_out, double* out,
                      int nthreads) {
  Problem p = make_problem(ORACLE_PASS);
  if (bad(p) || !bxy || n < 0) return -1;
  parallel_rows(n, nthreads, [&](int i) {
    const int b = bxy[3 * i], y = bxy[3 * i + 1], x = bxy[3 * i + 2];
    std::vector<double> beta(K), jc(C);
    if (J_out) {
      mlp_pixel(p, b, y, x, beta.data());
      blur_pixel(p, b, y, x, beta.data(), jc.data());
      for (int c = 0; c < C; ++c) J_out[(size_t)i * C + c] = jc[c];
    }
    if (out) {
      // memoised J (all channels) at the <= 4 distinct bilinear neighbours
      int ky[4], kx[4], nk = 0;
      std::vector<double> cache(4 * (size_t)C), bt(K);
      auto Jat = [&](int c, int yy, int xx) {
        for (int q = 0; q < nk; ++q)
          if (ky[q] == yy && kx[q] == xx) return cache[(size_t)q * C + c];
        mlp_pixel(p, b, yy, xx, bt.data());
        blur_pixel(p, b, yy, xx, bt.data(), &cache[(size_t)nk * C]);
        ky[nk] = yy; kx[nk] = xx;
        return cache[(size_t)(nk++) * C + c];
      };
      std::vector<double> o(C);
      warp_pixel(p, b, y, x, Jat, o.data());
      for (int c = 0; c < C; ++c) out[(size_t)i * C + c] = o[c];
    }
  });
  return 0;
}

// Warp alone on a given fp64 J [B][C][H][W] (pins step a3 independently of a1/a2).
int p2s_oracle_warp(const double* J, int B, int C, int H, int W, const float* tilt, double* out,
                    int nthreads) {
  if (!J || !out || B < 1 || C < 1 || H < 1 || W < 1) return -1;
  Problem p{};
  p.B = B; p.C = C; p.H = H; p.W = W; p.tilt = tilt;
  const size_t HW = (size_t)H * W;
  for (int b = 0; b < B; ++b) {
    auto Jat = [&](int c, int yy, int xx) {
      return J[((size_t)b * C + c) * HW + (size_t)yy * W + xx];
    };
    parallel_rows(H, nthreads, [&](int y) {
      std::vector<double> o(C);
      for (int x = 0; x < W; ++x) {
        warp_pixel(p, b, y, x, Jat, o.data());
        for (int c = 0; c < C; ++c) out[((size_t)b * C + c) * HW + (size_t)y * W + x] = o[c];
      }
    });
  }
  return 0;
}

// Anchor grid -> dense Zernike field (see the header): anchors [B][n_in][G][G] fp32,
// field [B][n_in][H][W] fp64 (rounded to fp32 by the caller when it feeds the render).
int p2s_oracle_interp_anchors(const float* anchors, int B, int n_in, int G, int H, int W, double* field) {
  if (!anchors || !field || B < 1 || n_in < 1 || G < 1 || H < 1 || W < 1) return -1;
  const size_t HW = (size_t)H * W, GG = (size_t)G * G;
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < n_in; ++k) {
      const float* A = anchors + ((size_t)b * n_in + k) * GG;
      double* F = field + ((size_t)b * n_in + k) * HW;
      for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
          if (G == 1) { F[(size_t)y * W + x] = A[0]; continue; }
          const double u = (y + 0.5) * (G - 1) / H, v = (x + 0.5) * (G - 1) / W;
          const int i0 = std::min((int)std::floor(u), G - 2), j0 = std::min((int)std::floor(v), G - 2);
          const double fy = u - i0, fx = v - j0;
          F[(size_t)y * W + x] = (1 - fy) * (1 - fx) * A[(size_t)i0 * G + j0] + (1 - fy) * fx * A[(size_t)i0 * G + j0 + 1] +
                                 fy * (1 - fx) * A[(size_t)(i0 + 1) * G + j0] + fy * fx * A[(size_t)(i0 + 1) * G + j0 + 1];
        }
    }
  return 0;
}

// Adjoint of step a2 (see the header) for beta [B][K][H][W] and gJ [B][C][H][W] (fp64):
// gbeta_out [B][K][H][W] and / or gimage_out [B][C][H][W] (fp64, either may be NULL). dL/dI is
// accumulated per thread in private frames (scatter order, no atomics) and then summed.
int p2s_oracle_adjoint_blur(const float* image, int B, int C, int H, int W, const float* taps, int K, int S,
                            const double* beta, const double* gJ, double* gbeta_out, double* gimage_out,
                            int nthreads) {
  if (!image || !taps || !beta || !gJ || B < 1 || C < 1 || H < 1 || W < 1 || K < 1 || S < 1 || (S % 2) == 0)
    return -1;
  const int r = (S - 1) / 2;
  const size_t HW = (size_t)H * W;
  nthreads = std::max(1, nthreads);
  for (int b = 0; b < B; ++b) {
    const double* bb = beta + (size_t)b * K * HW;
    const double* gj = gJ + (size_t)b * C * HW;
    if (gbeta_out)
      parallel_rows(H, nthreads, [&](int y) {
        std::vector<double> patch((size_t)S * S);
        for (int x = 0; x < W; ++x) {
          for (int k = 0; k < K; ++k) gbeta_out[((size_t)b * K + k) * HW + (size_t)y * W + x] = 0.0;
          for (int c = 0; c < C; ++c) {
            const float* img = image + ((size_t)b * C + c) * HW;
            for (int i = 0; i < S; ++i) {
              const int yy = clampi(y - (i - r), 0, H - 1);
              for (int j = 0; j < S; ++j) patch[(size_t)i * S + j] = img[(size_t)yy * W + clampi(x - (j - r), 0, W - 1)];
            }
            const double g = gj[(size_t)c * HW + (size_t)y * W + x];
            for (int k = 0; k < K; ++k) {
              const float* phi = taps + (size_t)k * S * S;
              double ck = 0.0;
              for (int t = 0; t < S * S; ++t) ck += (double)phi[t] * patch[t];
              gbeta_out[((size_t)b * K + k) * HW + (size_t)y * W + x] += g * ck;
            }
          }
        }
      });
    if (gimage_out) {
      std::vector<std::vector<double>> part(nthreads, std::vector<double>((size_t)C * HW, 0.0));
      std::vector<std::thread> th;
      std::atomic_int next{0};
      for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t]() {
          std::vector<double> h((size_t)S * S);
          double* acc = part[t].data();
          for (int y; (y = next.fetch_add(1)) < H;)
            for (int x = 0; x < W; ++x) {
              // h[i][j] = sum_k beta_k(y,x) phi_k[i][j]: the pixel's own PSF (Eq. 3/4)
              std::fill(h.begin(), h.end(), 0.0);
              for (int k = 0; k < K; ++k) {
                const double bk = bb[(size_t)k * HW + (size_t)y * W + x];
                const float* phi = taps + (size_t)k * S * S;
                for (int t2 = 0; t2 < S * S; ++t2) h[t2] += bk * (double)phi[t2];
              }
              for (int c = 0; c < C; ++c) {
                const double g = gj[(size_t)c * HW + (size_t)y * W + x];
                double* ac = acc + (size_t)c * HW;
                for (int i = 0; i < S; ++i) {
                  const int yy = clampi(y - (i - r), 0, H - 1);
                  for (int j = 0; j < S; ++j) ac[(size_t)yy * W + clampi(x - (j - r), 0, W - 1)] += h[(size_t)i * S + j] * g;
                }
              }
            }
        });
      for (auto& t : th) t.join();
      double* o = gimage_out + (size_t)b * C * HW;
      for (size_t e = 0; e < (size_t)C * HW; ++e) {
        double s = 0.0;
        for (int t = 0; t < nthreads; ++t) s += part[t][e];
        o[e] = s;
      }
    }
  }
  return 0;
}

}  // extern "C"
