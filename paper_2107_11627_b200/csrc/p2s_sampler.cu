// p2s_sampler.cu — correlated anchor-grid sampling, the step upstream of
// p2s_render_anchors (NEXT-1). PAPER.md:293-295 (Sec. 3.4): anchor coefficients "drawn from the
// correlation matrix", which "can be pre-computed". Stand-in covariance (reading N3;
// the Takato-formula parameters are not in the paper): separable over anchor row, anchor column
// and Zernike mode,
//     Cov[A_j(a,b), A_j'(a',b')] = R[j][j'] s(a-a') s(b-b'),  s(d) = exp(-d^2 / (2 l^2)) + 1e-6 [d=0]
// so a frame's anchors are A = (L_R (x) L_s (x) L_s) z with Cholesky factors computed once at
// init and z ~ N(0, I) drawn by a counter-based generator (any frame reproducible on its own):
// Philox4x32-10 (Salmon et al., SC'11), key = seed, counter = (frame, anchor, mode, 0),
// Box-Muller on the first two words. The sampler shares no code with oracle/sampler.py.
//
// Dense mode (p2s_sampler_init_dense; "a correlation matrix of size 64^2 x 64^2 =
// 4096 x 4096 which can be pre-computed ... 4096 sets of Zernike coefficients are drawn from the
// correlation matrix"): any SPD spatial correlation C over the G^2 anchors, A_f = (L_R (x) L) z_f
// with L = chol(C) computed once on the host (fp64, blocked, threaded). Per call the mode-mixed
// normals Y = z L_R^T (fp64, split into fp16 hi + lo) are drawn by k_draw_y and the product L Y is
// a tcgen05 GEMM (k_sample_dense): M = 128 anchors x N = 128 (frame, mode) columns per tile, K
// over the anchors of L's lower triangle only, three fp16 products per K-step, fp32 accumulation
// in TMEM: L_hi Y_hi into one accumulator, L_hi Y_lo' + L_lo' Y_hi into a second, where the lo
// parts are stored scaled by 2^11 (lo' = fp16((v - hi) 2^11): no subnormal lo parts) and L by
// 2^14 (entries down to ~4e-9 stay normal); the epilogue forms 2^-14 (D_hi + 2^-11 D_lo) --
// the dropped lo x lo term is ~2^-22 relative.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "p2s.h"
#include "sm100.cuh"

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = 0xD2511F53ull * c.x, p1 = 0xCD9E8D57ull * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double normal_at(uint32_t k0, uint32_t k1, uint32_t frame, uint32_t g, uint32_t j) {
  const uint4 x = philox4x32_10(make_uint4(frame, g, j, 0u), k0, k1);
  const double u1 = ((double)x.x + 0.5) * 0x1p-32, u2 = ((double)x.y + 0.5) * 0x1p-32;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

// One CTA per (mode j, frame f): Z'_j = sum_{j' <= j} L_R[j][j'] z_{j'} over the G x G anchors,
// then A_j = L_s Z'_j L_s^T (both triangular), all in fp64, stored fp32 [F][n_in][G][G].
__global__ void __launch_bounds__(256) k_sample_anchors(const double* __restrict__ Ls, const double* __restrict__ LR,
                                                        int G, int n_in, uint32_t k0, uint32_t k1, int frame0,
                                                        float* __restrict__ out) {
  extern __shared__ double sm[];
  double* Zp = sm;
  double* T = sm + G * G;
  const int j = blockIdx.x, f = blockIdx.y, GG = G * G;
  const uint32_t frame = (uint32_t)(frame0 + f);
  for (int g = threadIdx.x; g < GG; g += blockDim.x) {
    double acc = 0.0;
    for (int jp = 0; jp <= j; ++jp) acc += LR[j * n_in + jp] * normal_at(k0, k1, frame, (uint32_t)g, (uint32_t)jp);
    Zp[g] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < GG; e += blockDim.x) {  // T = L_s Z' (rows)
    const int a = e / G, b = e - a * G;
    double acc = 0.0;
    for (int c = 0; c <= a; ++c) acc += Ls[a * G + c] * Zp[c * G + b];
    T[e] = acc;
  }
  __syncthreads();
  float* o = out + ((size_t)f * n_in + j) * GG;
  for (int e = threadIdx.x; e < GG; e += blockDim.x) {  // A = T L_s^T (columns)
    const int a = e / G, b = e - a * G;
    double acc = 0.0;
    for (int d = 0; d <= b; ++d) acc += T[a * G + d] * Ls[b * G + d];
    o[e] = (float)acc;
  }
}

// in-place lower Cholesky of an n x n row-major SPD matrix (fp64); false if not positive definite
bool cholesky(std::vector<double>& A, int n) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      if (i == j) {
        if (!(s > 0.0)) return false;
        A[(size_t)i * n + i] = std::sqrt(s);
      } else {
        A[(size_t)i * n + j] = s / A[(size_t)j * n + j];
      }
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = 0.0;
  return true;
}

// ---------------------------------------------------------------- dense mode (tcgen05 GEMM)
// Operand tiles are stored pre-packed in the SWIZZLE_NONE K-major core-matrix layout, so one
// cp.async.bulk per operand lands a tile in shared memory ready for the UMMA descriptors:
// element (row, k) of a 128 x 64 fp16 tile at (row % 8) 16 + (row / 8) 1024 + (k % 8) 2 + (k / 8) 128
// bytes (LBO = 128 B along K, SBO = 1024 B along rows); a tile pair = [hi 16 KB | lo 16 KB].
constexpr int kDenseBM = 128, kDenseBN = 128, kDenseBK = 64;
constexpr int kDenseTile = kDenseBM * kDenseBK * 2;  // bytes of one fp16 tile
constexpr int kDensePair = 2 * kDenseTile;           // hi + lo
constexpr int kDenseStage = 2 * kDensePair;          // A pair + B pair
constexpr int kDenseStages = 3;
constexpr int kDenseThreads = 192;                   // w0 bulk-copy producer, w1 UMMA, w2-5 epilogue
constexpr int kDenseSmem = kDenseStages * kDenseStage + 256;
constexpr int kDenseMaxCols = 2048;                  // (frame, mode) columns per GEMM launch
constexpr double kDenseLScale = 16384.0;             // L stored x 2^14
constexpr double kDenseLoScale = 2048.0;             // lo parts stored x 2^11

__host__ __device__ __forceinline__ uint32_t core_off(int row, int k) {
  return (uint32_t)((row % 8) * 16 + (row / 8) * 1024 + (k % 8) * 2 + (k / 8) * 128);
}

struct DenseParams {
  const uint8_t* Lp;  // L tile pairs, lower block triangle: tile (mb, kb <= 2 mb + 1) at mb (mb + 1) + kb
  const uint8_t* Yp;  // Y tile pairs (nb, kb) at nb KB + kb
  float* out;         // anchors [frames][n_in][GG] of this launch's frames
  int GG, MB, NB, KB, ncols, n_in, ntiles;
};

// Y = z L_R^T for frames [frame0, frame0 + F), all anchors p < Np (zero for p >= G^2): block
// (anchor block of 128, frame); normals once per (p, k) into shared memory, then per thread (one
// anchor) the n_in mixed values, fp64, split into fp16 hi and lo' = fp16((y - hi) 2^11).
__global__ void __launch_bounds__(128) k_draw_y(const double* __restrict__ LR, int G, int n_in, uint32_t k0,
                                                uint32_t k1, int frame0, int KB, uint8_t* __restrict__ Yp) {
  extern __shared__ double zs[];  // [n_in][128]
  const int GG = G * G, p = blockIdx.x * 128 + threadIdx.x, f = blockIdx.y;
  const uint32_t frame = (uint32_t)(frame0 + f);
  for (int k = 0; k < n_in; ++k) zs[k * 128 + threadIdx.x] = p < GG ? normal_at(k0, k1, frame, (uint32_t)p, (uint32_t)k) : 0.0;
  __syncthreads();
  const int kb = p / kDenseBK, kk = p % kDenseBK;
  for (int j = 0; j < n_in; ++j) {
    double y = 0.0;
    for (int k = 0; k <= j; ++k) y += LR[j * n_in + k] * zs[k * 128 + threadIdx.x];
    const int n = f * n_in + j, nb = n / kDenseBN, row = n % kDenseBN;
    uint8_t* t = Yp + ((size_t)nb * KB + kb) * kDensePair + core_off(row, kk);
    const __half hi = __double2half(y);
    const __half lo = __double2half((y - (double)__half2float(hi)) * kDenseLoScale);
    *reinterpret_cast<__half*>(t) = hi;
    *reinterpret_cast<__half*>(t + kDenseTile) = lo;
  }
}

// A[p][(f, j)] = sum_q L[p][q] Y[q][(f, j)], persistent over (mb, nb) tiles, longest (largest mb)
// first; per tile two accumulators (hi x hi, and the two lo' products), TMEM double-buffered
// (2 x 256 columns) so one tile's epilogue overlaps the next tile's UMMAs.
__global__ void __launch_bounds__(kDenseThreads, 1) k_sample_dense(const DenseParams p) {
  using namespace p2s;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDenseStages * kDenseStage);
  uint64_t* empty = full + kDenseStages;
  uint64_t* acc_full = empty + kDenseStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDenseStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const int mb = p.MB - 1 - t / p.NB, nb = t % p.NB;
        for (int kb = 0; kb <= 2 * mb + 1; ++kb, ++it) {
          const int s = it % kDenseStages;
          mbar_wait(&empty[s], ((it / kDenseStages) & 1) ^ 1);
          uint8_t* dst = smem + s * kDenseStage;
          mbar_arrive_expect_tx(&full[s], kDenseStage);
          bulk_g2s(dst, p.Lp + ((size_t)mb * (mb + 1) + kb) * kDensePair, kDensePair, &full[s]);
          bulk_g2s(dst + kDensePair, p.Yp + ((size_t)nb * p.KB + kb) * kDensePair, kDensePair, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_f16(kDenseBM, kDenseBN);
    int it = 0, tl = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++tl) {
      const int mb = p.MB - 1 - t / p.NB;
      const int buf = tl & 1;
      mbar_wait(&acc_empty[buf], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(buf * 2 * kDenseBN), dlo = d + kDenseBN;
      for (int kb = 0; kb <= 2 * mb + 1; ++kb, ++it) {
        const int s = it % kDenseStages;
        mbar_wait(&full[s], (it / kDenseStages) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(smem + s * kDenseStage);
#pragma unroll
        for (int k16 = 0; k16 < kDenseBK / 16; ++k16) {
          const uint32_t o = base + (uint32_t)k16 * 256;
          const uint64_t ahi = sdesc(o, 128, 1024), alo = sdesc(o + kDenseTile, 128, 1024);
          const uint64_t bhi = sdesc(o + kDensePair, 128, 1024), blo = sdesc(o + kDensePair + kDenseTile, 128, 1024);
          const uint32_t acc = (kb | k16) != 0 ? 1u : 0u;
          umma_f16_elect(d, ahi, bhi, idesc, acc);
          umma_f16_elect(dlo, ahi, blo, idesc, acc);
          umma_f16_elect(dlo, alo, bhi, idesc, 1u);
        }
        umma_commit_elect(&empty[s]);  // the stage is free once these UMMAs have read it
      }
      umma_commit_elect(&acc_full[buf]);
    }
  } else {
    const int q = warp & 3, row = 32 * q + lane;
    int tl = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++tl) {
      const int mb = p.MB - 1 - t / p.NB, nb = t % p.NB;
      const int buf = tl & 1;
      mbar_wait(&acc_full[buf], (tl >> 1) & 1);
      tc_fence_after();
      const int a = mb * kDenseBM + row;
      const uint32_t tl_addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * 2 * kDenseBN);
      for (int cg = 0; cg < kDenseBN / 16; ++cg) {
        float v[16], w[16];
        tmem_ld16(tl_addr + (uint32_t)cg * 16, v);
        tmem_ld16(tl_addr + (uint32_t)(kDenseBN + cg * 16), w);
        tmem_ld_wait();
        if (a < p.GG) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = nb * kDenseBN + cg * 16 + i;
            // 2^-14 (D_hi + 2^-11 D_lo); n = f n_in + j: anchors [f][j][a]
            if (n < p.ncols) p.out[(size_t)n * p.GG + a] = fmaf(w[i], 0x1p-25f, v[i] * 0x1p-14f);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Lower Cholesky factor of an n x n row-major SPD matrix in place (fp64), right-looking with
// 64-column panels; the panel solve and the trailing update are split over host threads by
// rows. false if not positive definite.
bool cholesky_blocked(std::vector<double>& A, int n) {
  const int nb = 64;
  const int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto par_rows = [&](int r0, auto&& body) {
    if (n - r0 <= 0) return;
    std::vector<std::thread> th;
    const int use = std::min(nt, n - r0);
    for (int w = 0; w < use; ++w)
      th.emplace_back([&, w] {
        for (int i = r0 + w; i < n; i += use) body(i);
      });
    for (auto& t : th) t.join();
  };
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int k1 = std::min(n, k0 + nb);
    for (int i = k0; i < k1; ++i)  // diagonal block (earlier panels already subtracted)
      for (int j = k0; j <= i; ++j) {
        double s = A[(size_t)i * n + j];
        for (int k = k0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
        if (i == j) {
          if (!(s > 0.0)) return false;
          A[(size_t)i * n + i] = std::sqrt(s);
        } else {
          A[(size_t)i * n + j] = s / A[(size_t)j * n + j];
        }
      }
    par_rows(k1, [&](int i) {  // panel: rows below the diagonal block
      double* ai = &A[(size_t)i * n];
      for (int j = k0; j < k1; ++j) {
        const double* aj = &A[(size_t)j * n];
        double s = ai[j];
        for (int k = k0; k < j; ++k) s -= ai[k] * aj[k];
        ai[j] = s / aj[j];
      }
    });
    par_rows(k1, [&](int i) {  // trailing update of row i, columns [k1, i]
      double* ai = &A[(size_t)i * n];
      for (int j = k1; j <= i; ++j) {
        const double* aj = &A[(size_t)j * n];
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        int k = k0;
        for (; k + 4 <= k1; k += 4) {
          s0 += ai[k] * aj[k];
          s1 += ai[k + 1] * aj[k + 1];
          s2 += ai[k + 2] * aj[k + 2];
          s3 += ai[k + 3] * aj[k + 3];
        }
        for (; k < k1; ++k) s0 += ai[k] * aj[k];
        ai[j] -= (s0 + s1) + (s2 + s3);
      }
    });
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = 0.0;
  return true;
}

bool mode_factor(int n_in, const double* mode_cov, std::vector<double>& R) {
  R.assign((size_t)n_in * n_in, 0.0);
  for (int i = 0; i < n_in; ++i)
    for (int j = 0; j < n_in; ++j)
      R[(size_t)i * n_in + j] = mode_cov ? mode_cov[(size_t)i * n_in + j] : (i == j ? 0.25 : 0.0);
  for (int i = 0; i < n_in; ++i)
    for (int j = 0; j < i; ++j)
      if (R[(size_t)i * n_in + j] != R[(size_t)j * n_in + i]) return false;  // not symmetric
  return cholesky(R, n_in);
}

}  // namespace

struct p2s_sampler {
  int G = 0, n_in = 0;
  double* d_Ls = nullptr;
  double* d_LR = nullptr;
  // dense mode
  int dense = 0, Np = 0, MB = 0, KB = 0, sm_count = 0;
  uint8_t* d_Lp = nullptr;
  uint8_t* d_Yp = nullptr;
};

extern "C" {

p2s_status p2s_sampler_init(int G, int n_in, double corr_len, const double* mode_cov, p2s_sampler** out) {
  if (!out || G < 1 || G > 64 || n_in < 1 || n_in > 64 || !(corr_len >= 0.0)) return P2S_ERR_INVALID_ARG;
  *out = nullptr;
  std::vector<double> S((size_t)G * G), R;
  for (int a = 0; a < G; ++a)
    for (int c = 0; c < G; ++c) {
      const double d = (double)(a - c);
      S[(size_t)a * G + c] = (corr_len > 0.0 ? std::exp(-d * d / (2.0 * corr_len * corr_len)) : (a == c ? 1.0 : 0.0)) +
                             (a == c ? 1e-6 : 0.0);
    }
  if (!cholesky(S, G) || !mode_factor(n_in, mode_cov, R)) return P2S_ERR_INVALID_ARG;  // not SPD
  if (cudaFuncSetAttribute(k_sample_anchors, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * 64 * 64 * (int)sizeof(double)) != cudaSuccess)
    return P2S_ERR_CUDA;
  p2s_sampler* s = new (std::nothrow) p2s_sampler();
  if (!s) return P2S_ERR_OOM;
  s->G = G;
  s->n_in = n_in;
  if (cudaMalloc(&s->d_Ls, S.size() * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&s->d_LR, R.size() * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(s->d_Ls, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(s->d_LR, R.data(), R.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    p2s_sampler_destroy(s);
    return P2S_ERR_CUDA;
  }
  *out = s;
  return P2S_OK;
}

p2s_status p2s_sampler_init_dense(int G, int n_in, const double* spatial_cov, int is_factor, const double* mode_cov,
                                  p2s_sampler** out) {
  if (!out || !spatial_cov || G < 1 || G > 64 || n_in < 1 || n_in > 64) return P2S_ERR_INVALID_ARG;
  *out = nullptr;
  const int GG = G * G;
  std::vector<double> L(spatial_cov, spatial_cov + (size_t)GG * GG), R;
  if (is_factor) {
    for (int i = 0; i < GG; ++i) {
      if (!(L[(size_t)i * GG + i] > 0.0)) return P2S_ERR_INVALID_ARG;
      for (int j = i + 1; j < GG; ++j) L[(size_t)i * GG + j] = 0.0;
    }
  } else {
    for (int i = 0; i < GG; ++i)
      for (int j = 0; j < i; ++j)
        if (L[(size_t)i * GG + j] != L[(size_t)j * GG + i]) return P2S_ERR_INVALID_ARG;  // not symmetric
    if (!cholesky_blocked(L, GG)) return P2S_ERR_INVALID_ARG;  // not positive definite
  }
  if (!mode_factor(n_in, mode_cov, R)) return P2S_ERR_INVALID_ARG;
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return P2S_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return P2S_ERR_UNSUPPORTED;
  // pack L's lower block triangle as fp16 hi / lo tile pairs (zero beyond G^2)
  const int Np = (GG + kDenseBM - 1) / kDenseBM * kDenseBM, MB = Np / kDenseBM, KB = Np / kDenseBK;
  std::vector<uint8_t> Lp((size_t)MB * (MB + 1) * kDensePair, 0);
  for (int mb = 0; mb < MB; ++mb)
    for (int kb = 0; kb <= 2 * mb + 1; ++kb) {
      uint8_t* t = Lp.data() + ((size_t)mb * (mb + 1) + kb) * kDensePair;
      for (int r = 0; r < kDenseBM; ++r)
        for (int k = 0; k < kDenseBK; ++k) {
          const int i = mb * kDenseBM + r, j = kb * kDenseBK + k;
          if (i >= GG || j >= GG || j > i) continue;
          const double v = L[(size_t)i * GG + j] * kDenseLScale;
          const __half hi = __double2half(v), lo = __double2half((v - (double)__half2float(hi)) * kDenseLoScale);
          std::memcpy(t + core_off(r, k), &hi, 2);
          std::memcpy(t + kDenseTile + core_off(r, k), &lo, 2);
        }
    }
  if (cudaFuncSetAttribute(k_sample_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseSmem) != cudaSuccess ||
      cudaFuncSetAttribute(k_draw_y, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 128 * 8) != cudaSuccess)
    return P2S_ERR_CUDA;
  p2s_sampler* s = new (std::nothrow) p2s_sampler();
  if (!s) return P2S_ERR_OOM;
  s->G = G;
  s->n_in = n_in;
  s->dense = 1;
  s->Np = Np;
  s->MB = MB;
  s->KB = KB;
  s->sm_count = prop.multiProcessorCount;
  const int nb_max = (std::max(n_in, kDenseMaxCols / n_in * n_in) + kDenseBN - 1) / kDenseBN;
  const size_t ybytes = (size_t)nb_max * KB * kDensePair;
  if (cudaMalloc(&s->d_LR, R.size() * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(s->d_LR, R.data(), R.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&s->d_Lp, Lp.size()) != cudaSuccess ||
      cudaMemcpy(s->d_Lp, Lp.data(), Lp.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&s->d_Yp, ybytes) != cudaSuccess || cudaMemset(s->d_Yp, 0, ybytes) != cudaSuccess) {
    p2s_sampler_destroy(s);
    return P2S_ERR_OOM;
  }
  *out = s;
  return P2S_OK;
}

p2s_status p2s_sample_anchors(p2s_sampler* s, unsigned long long seed, int frame0, int F, float* anchors,
                              p2s_stream_t stream) {
  if (!s || !anchors || F < 1 || F > 65535 || frame0 < 0) return P2S_ERR_INVALID_ARG;
  if (s->dense) {
    const int GG = s->G * s->G, fc = std::max(1, kDenseMaxCols / s->n_in);
    const uint32_t k0 = (uint32_t)(seed & 0xffffffffull), k1 = (uint32_t)(seed >> 32);
    for (int f0 = 0; f0 < F; f0 += fc) {
      const int nf = std::min(fc, F - f0);
      k_draw_y<<<dim3((unsigned)(s->Np / 128), (unsigned)nf), 128, (size_t)s->n_in * 128 * 8, (cudaStream_t)stream>>>(
          s->d_LR, s->G, s->n_in, k0, k1, frame0 + f0, s->KB, s->d_Yp);
      DenseParams p{};
      p.Lp = s->d_Lp;
      p.Yp = s->d_Yp;
      p.out = anchors + (size_t)f0 * s->n_in * GG;
      p.GG = GG;
      p.MB = s->MB;
      p.KB = s->KB;
      p.ncols = nf * s->n_in;
      p.NB = (p.ncols + kDenseBN - 1) / kDenseBN;
      p.n_in = s->n_in;
      p.ntiles = p.MB * p.NB;
      k_sample_dense<<<std::min(p.ntiles, s->sm_count), kDenseThreads, kDenseSmem, (cudaStream_t)stream>>>(p);
    }
    return cudaPeekAtLastError() == cudaSuccess ? P2S_OK : P2S_ERR_CUDA;
  }
  const size_t smem = 2 * (size_t)s->G * s->G * sizeof(double);
  k_sample_anchors<<<dim3((unsigned)s->n_in, (unsigned)F), 256, smem, (cudaStream_t)stream>>>(
      s->d_Ls, s->d_LR, s->G, s->n_in, (uint32_t)(seed & 0xffffffffull), (uint32_t)(seed >> 32), frame0, anchors);
  return cudaPeekAtLastError() == cudaSuccess ? P2S_OK : P2S_ERR_CUDA;
}

void p2s_sampler_destroy(p2s_sampler* s) {
  if (!s) return;
  cudaFree(s->d_Ls);
  cudaFree(s->d_LR);
  cudaFree(s->d_Lp);
  cudaFree(s->d_Yp);
  delete s;
}

}  // extern "C"
