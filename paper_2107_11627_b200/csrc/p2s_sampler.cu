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
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <new>
#include <vector>

#include "p2s.h"

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

}  // namespace

struct p2s_sampler {
  int G = 0, n_in = 0;
  double* d_Ls = nullptr;
  double* d_LR = nullptr;
};

extern "C" {

p2s_status p2s_sampler_init(int G, int n_in, double corr_len, const double* mode_cov, p2s_sampler** out) {
  if (!out || G < 1 || G > 64 || n_in < 1 || n_in > 64 || !(corr_len >= 0.0)) return P2S_ERR_INVALID_ARG;
  *out = nullptr;
  std::vector<double> S((size_t)G * G), R((size_t)n_in * n_in, 0.0);
  for (int a = 0; a < G; ++a)
    for (int c = 0; c < G; ++c) {
      const double d = (double)(a - c);
      S[(size_t)a * G + c] = (corr_len > 0.0 ? std::exp(-d * d / (2.0 * corr_len * corr_len)) : (a == c ? 1.0 : 0.0)) +
                             (a == c ? 1e-6 : 0.0);
    }
  for (int i = 0; i < n_in; ++i)
    for (int j = 0; j < n_in; ++j)
      R[(size_t)i * n_in + j] = mode_cov ? mode_cov[(size_t)i * n_in + j] : (i == j ? 0.25 : 0.0);
  for (int i = 0; i < n_in; ++i)
    for (int j = 0; j < i; ++j)
      if (R[(size_t)i * n_in + j] != R[(size_t)j * n_in + i]) return P2S_ERR_INVALID_ARG;  // not symmetric
  if (!cholesky(S, G) || !cholesky(R, n_in)) return P2S_ERR_INVALID_ARG;  // not positive definite
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

p2s_status p2s_sample_anchors(p2s_sampler* s, unsigned long long seed, int frame0, int F, float* anchors,
                              p2s_stream_t stream) {
  if (!s || !anchors || F < 1 || F > 65535 || frame0 < 0) return P2S_ERR_INVALID_ARG;
  const size_t smem = 2 * (size_t)s->G * s->G * sizeof(double);
  k_sample_anchors<<<dim3((unsigned)s->n_in, (unsigned)F), 256, smem, (cudaStream_t)stream>>>(
      s->d_Ls, s->d_LR, s->G, s->n_in, (uint32_t)(seed & 0xffffffffull), (uint32_t)(seed >> 32), frame0, anchors);
  return cudaPeekAtLastError() == cudaSuccess ? P2S_OK : P2S_ERR_CUDA;
}

void p2s_sampler_destroy(p2s_sampler* s) {
  if (!s) return;
  cudaFree(s->d_Ls);
  cudaFree(s->d_LR);
  delete s;
}

}  // extern "C"
