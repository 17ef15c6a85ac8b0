// p2s_anchor.cu — the anchor-grid interpolation as a standalone op and its adjoint (SURVEY
// §8(f) NEXT-1 with NEXT-4: the paper's own input path, "anchor points ...
// interpolated", made differentiable). Registration (reading N1): pixel
// centre (t + 0.5), anchors at a n / (G - 1); per mode
//     z[y][x] = sum_{a,b} wy[y][a] wx[x][b] A[a][b]        (bilinear, separable: z = Wy A Wx^T)
//     dL/dA[a][b] = sum_{y,x} wy[y][a] wx[x][b] dL/dz[y][x]   (dL/dA = Wy^T dL/dz Wx)
// with u = (t + 0.5)(G - 1)/n, i0 = min(floor(u), G - 2), weights 1 - (u - i0) on i0 and
// u - i0 on i0 + 1, computed in fp32 exactly as the fused kernel's anchor staging
// (p2s_kernels.cuh build_A1_anchors), so that p2s_render on p2s_interp_anchors' field
// reproduces p2s_render_anchors. Memory-bound SIMT kernels (no contraction to put on tensor
// cores: 4 weights per pixel).
#include <cuda_runtime.h>

#include <cstdint>

#include "p2s.h"

namespace {

struct Lin { int i0; float f; };

// the fused kernel's fp32 formula (build_A1_anchors)
__device__ __forceinline__ Lin lin(int t, int G, int n) {
  if (G <= 1) return Lin{0, 0.f};
  const float u = (t + 0.5f) * (float)(G - 1) / (float)n;
  const int i0 = min((int)floorf(u), G - 2);
  return Lin{i0, u - (float)i0};
}

// weight of anchor a for pixel index t (0 outside its two anchors)
__device__ __forceinline__ float wgt(int t, int a, int G, int n) {
  if (G <= 1) return 1.f;
  const Lin l = lin(t, G, n);
  return l.i0 == a ? 1.f - l.f : (l.i0 + 1 == a ? l.f : 0.f);
}

// z[b][k][y][x]: R_j = (1 - fy) A[i0][j] + fy A[i0 + 1][j], then (1 - fx) R_j0 + fx R_j0+1 — the
// order and grouping of build_A1_anchors' separable path
__global__ void __launch_bounds__(256) k_interp_anchors(const float* __restrict__ A, int B, int n_in, int G, int H,
                                                        int W, float* __restrict__ z) {
  const size_t HW = (size_t)H * W, n = (size_t)B * n_in * HW;
  const int di = G > 1 ? G : 0, dj = G > 1 ? 1 : 0;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const size_t plane = e / HW, r = e - plane * HW;
    const int y = (int)(r / W), x = (int)(r - (size_t)y * W);
    const Lin ly = lin(y, G, H), lx = lin(x, G, W);
    const float* a = A + plane * (size_t)G * G + (size_t)ly.i0 * G + lx.i0;
    const float r0 = (1.f - ly.f) * __ldg(a) + ly.f * __ldg(a + di);
    const float r1 = (1.f - ly.f) * __ldg(a + dj) + ly.f * __ldg(a + di + dj);
    z[e] = (1.f - lx.f) * r0 + lx.f * r1;
  }
}

// one warp per anchor (b, k, a, c): dL/dA[a][c] = sum over its support rectangle of
// wy(y, a) wx(x, c) dL/dz[y][x]; lanes stride the support columns, a fixed shuffle tree reduces
// (deterministic). The support is found conservatively and the weights decide exactly.
__global__ void __launch_bounds__(256) k_anchors_backward(const float* __restrict__ gz, int B, int n_in, int G, int H,
                                                          int W, float* __restrict__ gA) {
  const int lane = threadIdx.x & 31;
  const size_t nwarps = (size_t)B * n_in * G * G;
  const size_t HW = (size_t)H * W;
  for (size_t wi = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nwarps;
       wi += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const size_t plane = wi / ((size_t)G * G);
    const int rem = (int)(wi - plane * G * G), a = rem / G, c = rem - a * G;
    int y0 = 0, y1 = H - 1, x0 = 0, x1 = W - 1;
    if (G > 1) {  // anchor a is used by pixels with u in (a - 1, a + 1) (or beyond at the ends)
      const float sy = (float)H / (float)(G - 1), sx = (float)W / (float)(G - 1);
      y0 = a <= 1 ? 0 : max(0, (int)floorf((a - 1) * sy - 0.5f) - 1);
      y1 = a >= G - 2 ? H - 1 : min(H - 1, (int)ceilf((a + 1) * sy - 0.5f) + 1);
      x0 = c <= 1 ? 0 : max(0, (int)floorf((c - 1) * sx - 0.5f) - 1);
      x1 = c >= G - 2 ? W - 1 : min(W - 1, (int)ceilf((c + 1) * sx - 0.5f) + 1);
    }
    const float* g = gz + plane * HW;
    float acc = 0.f;
    for (int y = y0; y <= y1; ++y) {
      const float wy = wgt(y, a, G, H);
      if (wy == 0.f) continue;
      const float* gr = g + (size_t)y * W;
      float s = 0.f;
      for (int x = x0 + lane; x <= x1; x += 32) s += wgt(x, c, G, W) * __ldg(gr + x);
      acc += wy * s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) gA[wi] = acc;
  }
}

int grid_for(size_t work, int per_block) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t blocks = (work + per_block - 1) / per_block;
  return (int)(blocks < (size_t)sms * 16 ? (blocks ? blocks : 1) : (size_t)sms * 16);
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char *pa = (const char*)a, *pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

}  // namespace

extern "C" {

p2s_status p2s_interp_anchors(const float* anchors, int B, int n_in, int G, int H, int W, float* zernike_field,
                              p2s_stream_t stream) {
  if (!anchors || !zernike_field || B < 1 || n_in < 1 || G < 1 || G > 4096 || H < 1 || W < 1)
    return P2S_ERR_INVALID_ARG;
  const size_t nz = (size_t)B * n_in * H * W, na = (size_t)B * n_in * G * G;
  if (overlaps(zernike_field, nz * 4, anchors, na * 4)) return P2S_ERR_INVALID_ARG;
  k_interp_anchors<<<grid_for(nz, 256), 256, 0, (cudaStream_t)stream>>>(anchors, B, n_in, G, H, W, zernike_field);
  return cudaPeekAtLastError() == cudaSuccess ? P2S_OK : P2S_ERR_CUDA;
}

p2s_status p2s_anchors_backward(const float* grad_zernike, int B, int n_in, int G, int H, int W, float* grad_anchors,
                                p2s_stream_t stream) {
  if (!grad_zernike || !grad_anchors || B < 1 || n_in < 1 || G < 1 || G > 4096 || H < 1 || W < 1)
    return P2S_ERR_INVALID_ARG;
  const size_t nz = (size_t)B * n_in * H * W, na = (size_t)B * n_in * G * G;
  if (overlaps(grad_anchors, na * 4, grad_zernike, nz * 4)) return P2S_ERR_INVALID_ARG;
  k_anchors_backward<<<grid_for(na * 32, 256), 256, 0, (cudaStream_t)stream>>>(grad_zernike, B, n_in, G, H, W,
                                                                               grad_anchors);
  return cudaPeekAtLastError() == cudaSuccess ? P2S_OK : P2S_ERR_CUDA;
}

}  // extern "C"
