// conv_probe.cu — 2-CTA UMMA throughput for the fused kernel's convolution walk (dev tool, not
// product code). Replays the K-step descriptor sequence of the S=33 plan (V16 EY views + H rows,
// 3 channels sharing each B slab) against fixed-descriptor and ring-walk variants, and reports
// cycles per UMMA (M=256, N=112, floor 56).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace p2s;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kSteps = 69;          // S=33: 66 V16 steps + 3 H steps
constexpr uint32_t kYStride = 2624; // EY block stride (164 positions x 16 B)
constexpr uint32_t kChan = 13312;   // bytes per channel of E views (rounded)
constexpr uint32_t kSlab = 1792;    // one CTA's half of a B slab (56 rows x 32 B)
constexpr int kRingSlabs = 27;      // 3 stages x 9 slabs

struct Step { uint32_t off, lbo; };

// A_MODE 0: four fixed nearby descriptors; 1: the real K-step walk.
// B_MODE 0: four rotating slabs; 1: walk through the ring.
// CH: UMMAs per K-step (channels sharing a B slab). COMMIT: commit every 9 K-steps (per item).
template <int A_MODE, int B_MODE, int CH, int COMMIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_conv(const Step* steps_g, int reps, unsigned long long* cyc, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  __shared__ uint32_t sSteps[kSteps];
  // fill 0: zeros; 1: random fp16 in [-0.5, 0.5) (what the kernel multiplies)
  for (int i = threadIdx.x * 16; i < 160 * 1024; i += 128 * 16) {
    uint32_t w[4];
    for (int q = 0; q < 4; ++q) {
      uint32_t h = (uint32_t)(i + 4 * q) * 2654435761u + blockIdx.x * 40503u;
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      const float a = (float)(h & 0xffff) / 65536.f - 0.5f, c = (float)(h >> 16) / 65536.f - 0.5f;
      w[q] = fill ? pack_half2(a, c) : 0u;
    }
    *reinterpret_cast<int4*>(smem + i) = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
  }
  for (int i = threadIdx.x; i < kSteps; i += 128) sSteps[i] = (steps_g[i].off >> 4) | ((steps_g[i].lbo >> 4) << 16);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool leader = cluster_ctarank() == 0;
  if (warp_id() == 0 && leader) {
    const uint32_t id = idesc_f16(256, 112);
    const uint32_t e_lo = smem_u32(smem) >> 4;
    const uint32_t ring_lo = (smem_u32(smem + 64 * 1024) >> 4) | ((128u >> 4) << 16);
    const uint32_t hi_a = (128u >> 4) | (1u << 14), hi_b = (256u >> 4) | (1u << 14);
    const uint32_t ch16 = kChan >> 4;
    long long t0 = clock64();
    uint32_t slab = 0;
    int n = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 2
      for (int t = 0; t < kSteps; ++t) {
        uint32_t a_lo;
        if (A_MODE == 0) a_lo = e_lo + (5u * (t & 3)) | ((kYStride >> 4) << 16);
        else a_lo = e_lo + sSteps[t];
        uint32_t b_lo;
        if (B_MODE == 0) b_lo = ring_lo + (t & 3) * (kSlab >> 4);
        else b_lo = ring_lo + slab * (kSlab >> 4);
        if (++slab == kRingSlabs) slab = 0;
        const uint64_t bd = ((uint64_t)hi_b << 32) | b_lo;
#pragma unroll
        for (int c = 0; c < CH; ++c)
          umma2_f16_elect(tmem + c * 112, ((uint64_t)hi_a << 32) | (a_lo + c * ch16), bd, id, t > 0);
        if (COMMIT == 1 && ++n == 9) { n = 0; umma2_commit_elect(&bar); }
        if (COMMIT == 2 && ++n == 11) {  // the kernel's per-item control path
          n = 0;
          umma2_commit_elect(&bar);
          mbar_wait(&bar2, 1);          // already-complete phase: a probe round trip
          tc_fence_after();
        }
      }
    }
    umma2_commit_elect(&bar2);
    mbar_wait(&bar2, 0);
    long long t1 = clock64();
    if (lane_id() == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<512>(tmem);
}

// Queue depth: per-UMMA issue timestamps from an idle pipe (issue stalls once the queue is full).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_qdepth(unsigned long long* ts) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 160 * 1024; i += 128 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp_id() == 0 && cluster_ctarank() == 0) {
    const uint32_t id = idesc_f16(256, 112);
    const uint64_t ad = sdesc(smem_u32(smem), 2624, 128), bd = sdesc(smem_u32(smem + 64 * 1024), 128, 256);
    long long t[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      umma2_f16_elect(tmem + (j % 3) * 112, ad, bd, id, 1);
      t[j] = clock64();
    }
    umma2_commit_elect(&bar);
    mbar_wait(&bar, 0);
    const long long te = clock64();
    if (lane_id() == 0 && blockIdx.x == 0) {
      for (int j = 0; j < 64; ++j) ts[j] = (unsigned long long)(t[j] - t[0]);
      ts[64] = (unsigned long long)(te - t[0]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<512>(tmem);
}

// Accumulator dependency: UMMAs (M=256, width N) rotating over NACC independent accumulators,
// A descriptor fixed or walking (16-B steps, like the conv / MLP K-loops).
template <int N, int NACC, bool WALK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_dep(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 160 * 1024; i += 128 * 16) {
    const uint32_t h = (uint32_t)i * 2654435761u;
    *reinterpret_cast<int4*>(smem + i) = make_int4((int)(h & 0x3bff3bff), (int)((h >> 3) & 0x3bff3bff), 0, 0);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp_id() == 0 && cluster_ctarank() == 0) {
    const uint32_t id = idesc_f16(256, N);
    const uint32_t a0 = smem_u32(smem) >> 4, b0 = (smem_u32(smem + 96 * 1024) >> 4) | ((128u >> 4) << 16);
    const uint32_t hi_a = (3328u >> 4) | (1u << 14), hi_b = (256u >> 4) | (1u << 14);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int acc = it % NACC;
      const uint32_t alo = (a0 + (WALK ? (uint32_t)(it % 13) * 16u : 0u)) | ((128u >> 4) << 16);
      const uint32_t blo = b0 + (uint32_t)(it % 13) * (uint32_t)(N * 16 / 16);
      umma2_f16_elect(tmem + acc * 128, ((uint64_t)hi_a << 32) | alo, ((uint64_t)hi_b << 32) | blo, id, 1);
    }
    umma2_commit_elect(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<512>(tmem);
}
template <int N, int NACC, bool WALK>
static void run_dep(int nsm) {
  unsigned long long* dc; CK(cudaMalloc(&dc, 1024 * 8)); CK(cudaMemset(dc, 0, 1024 * 8));
  auto k = k_dep<N, NACC, WALK>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  const int iters = 3900;
  for (int w = 0; w < 2; ++w) { k<<<nsm, 128, 160 * 1024>>>(iters, dc); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
  std::vector<unsigned long long> c(nsm);
  CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double mean = 0; int nl = 0;
  for (int i = 0; i < nsm; i += 2) { mean += c[i]; ++nl; }
  printf("dep N=%3d accumulators=%d A=%s: %.1f cyc/UMMA (floor %d)\n", N, NACC, WALK ? "walk " : "fixed",
         mean / nl / iters, N / 2);
  cudaFree(dc);
}

// TMEM -> register bandwidth: NW warps (quadrant = warp % 4), each loading NL x (32 lanes x
// X columns) per tcgen05.wait::ld, for `iters` rounds over 448 columns.
template <int X>
__device__ __forceinline__ void tld(uint32_t a, float* v) {
  if constexpr (X == 16) tmem_ld16(a, *reinterpret_cast<float(*)[16]>(v));
  else if constexpr (X == 8) tmem_ld8(a, v);
  else tmem_ld4(a, v);
}
template <int X, int NL>
__global__ void __launch_bounds__(512, 1) k_tmem_bw(int nw, int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t tslot;
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int w = warp_id();
  float acc8[X];
#pragma unroll
  for (int i = 0; i < X; ++i) acc8[i] = 0.f;
  long long t0 = clock64();
  if (w < nw) {
    const uint32_t tl = tmem + ((uint32_t)((w & 3) * 32) << 16);
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c + NL * X <= 448; c += NL * X) {
        float v[NL][X];
#pragma unroll
        for (int l = 0; l < NL; ++l) tld<X>(tl + c + l * X, v[l]);
        tmem_ld_wait();
#pragma unroll
        for (int l = 0; l < NL; ++l)
#pragma unroll
          for (int i = 0; i < X; ++i) acc8[i] += v[l][i];  // independent chains
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = (unsigned long long)(clock64() - t0);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < X; ++i) acc += acc8[i];
  sink[threadIdx.x] = acc + (float)(t1 - t0) * 0.f;
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}
template <int X, int NL>
static void run_tmem_bw(int nw) {
  unsigned long long* dc; float* sink; CK(cudaMalloc(&dc, 8)); CK(cudaMalloc(&sink, 512 * 4));
  const int iters = 200;
  for (int w = 0; w < 2; ++w) { k_tmem_bw<X, NL><<<1, 512>>>(nw, iters, dc, sink); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
  unsigned long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
  const int per = 448 / (NL * X) * (NL * X);
  const double bytes = (double)iters * per * 32 * 4 * nw;
  printf("tmem ld x%-2d x %d per wait, %2d warps: %.1f B/cyc\n", X, NL, nw, bytes / c);
  cudaFree(dc); cudaFree(sink);
}

template <int A, int B, int CH, int COMMIT>
static void run(int nsm, const Step* d_steps, int fill = 0) {
  unsigned long long* dc; CK(cudaMalloc(&dc, 1024 * 8)); CK(cudaMemset(dc, 0, 1024 * 8));
  auto k = k_conv<A, B, CH, COMMIT>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  const int reps = 40;
  for (int w = 0; w < 2; ++w) { k<<<nsm, 128, 160 * 1024>>>(d_steps, reps, dc, fill); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
  std::vector<unsigned long long> c(nsm);
  CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double mx = 0, mean = 0; int nl = 0;
  for (int i = 0; i < nsm; i += 2) { mx = fmax(mx, (double)c[i]); mean += c[i]; ++nl; }
  const double per = (double)reps * kSteps * CH;
  printf("A=%s B=%s ch=%d commit=%d data=%s: %.1f cyc/UMMA mean, %.1f max (floor 56)\n", A ? "walk " : "fixed",
         B ? "ring " : "fixed", CH, COMMIT, fill ? "random" : "zeros ", mean / nl / per, mx / per);
  cudaFree(dc);
}

int main() {
  // S=33 plan: V16 steps (g, b): off = 2g*ystride + b*16, LBO = ystride; H steps p: EX row at
  // xbase = 4*ystride, off = xbase + 16*16*p, LBO = 128.
  std::vector<Step> st;
  for (int g = 0; g < 2; ++g)
    for (int b = 0; b < 33; ++b) st.push_back({2u * g * kYStride + b * 16u, kYStride});
  for (int p = 0; p < 3; ++p) st.push_back({4u * kYStride + 256u * p, 128u});
  Step* d; CK(cudaMalloc(&d, st.size() * sizeof(Step)));
  CK(cudaMemcpy(d, st.data(), st.size() * sizeof(Step), cudaMemcpyHostToDevice));
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  run<1, 1, 3, 1>(nsm, d, 1);
  run<1, 1, 3, 2>(nsm, d, 1);
  run<0, 0, 3, 0>(nsm, d, 1);
  run<0, 0, 3, 0>(nsm, d);
  run<1, 0, 3, 0>(nsm, d);
  run<0, 1, 3, 0>(nsm, d);
  run<1, 1, 3, 0>(nsm, d);
  run<1, 1, 3, 1>(nsm, d);
  run<1, 1, 1, 0>(nsm, d);
  run<0, 0, 1, 0>(nsm, d);
  {
    unsigned long long* dt; CK(cudaMalloc(&dt, 65 * 8));
    CK(cudaFuncSetAttribute(k_qdepth, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    for (int w = 0; w < 2; ++w) { k_qdepth<<<2, 128, 160 * 1024>>>(dt); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
    unsigned long long h[65]; CK(cudaMemcpy(h, dt, 65 * 8, cudaMemcpyDeviceToHost));
    printf("issue timestamps (cycles since 1st UMMA):");
    for (int j = 0; j < 64; ++j) printf("%s%llu", j % 16 ? " " : "\n  ", h[j]);
    printf("\n  all 64 complete at %llu\n", h[64]);
  }
  run_dep<80, 1, false>(nsm); run_dep<80, 1, true>(nsm); run_dep<80, 2, true>(nsm); run_dep<80, 3, true>(nsm);
  run_dep<112, 1, false>(nsm); run_dep<112, 1, true>(nsm); run_dep<112, 2, true>(nsm); run_dep<112, 3, true>(nsm);
  run_dep<128, 1, true>(nsm); run_dep<128, 2, true>(nsm);
  run_dep<208, 1, true>(nsm); run_dep<208, 2, true>(nsm);
  printf("PROBE DONE\n");
  return 0;
}
