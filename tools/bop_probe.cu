// bop_probe.cu — microbenchmark: what a conv UMMA (N = 112, K = 16, overlapped A views) costs as a
// function of how often its B operand changes and how many accumulators the stream rotates over
// (not product code; a development tool). The three-channel tile issues 3 UMMAs per B slab into
// 3 accumulators; the one-channel tile 1 UMMA per B slab into 1 accumulator.
//   pair  : cta_group::2, M = 256, B half per CTA (the fused kernel's form)
//   single: cta_group::1, M = 128, the whole B slab in this CTA's shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace p2s;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kNB = 16;  // distinct B slabs cycled through (a ring stage's worth)

// BPS: UMMAs per B slab; NACC: accumulators rotated over; ASTEP: 1 = consecutive UMMAs read A views
// 16 B apart (the conv walk), 0 = the same A view
template <int BPS, int NACC, int ASTEP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 128 * 1024; i += 128 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  uint32_t tmem = tslot;
  const bool leader = cluster_ctarank() == 0;
  if (warp_id() == 0 && leader) {
    constexpr uint32_t id = idesc_f16(256, 112);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int slab = (it / BPS) % kNB, j = it % BPS;
      const uint64_t ad = sdesc(sa + (ASTEP ? ((it / BPS) % 32) * 16 : 0) + (j % 3) * 2624 * 8, 2624, 128);
      const uint64_t bd = sdesc(sb + slab * 2048, 128, 256);  // this CTA's half: 56 rows x 16 fp16 = 1792 B
      umma2_f16_elect(tmem + (it % NACC) * 112, ad, bd, id, 1);
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

template <int BPS, int NACC, int ASTEP>
__global__ void __launch_bounds__(128, 1) k_single(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 128 * 1024; i += 128 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tslot;
  if (warp_id() == 0) {
    constexpr uint32_t id = idesc_f16(128, 112);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int slab = (it / BPS) % kNB, j = it % BPS;
      const uint64_t ad = sdesc(sa + (ASTEP ? ((it / BPS) % 32) * 16 : 0) + (j % 3) * 2624 * 8, 2624, 128);
      const uint64_t bd = sdesc(sb + slab * 4096, 128, 256);  // the whole slab: 112 rows x 16 fp16 = 3584 B
      if (lane_id() == 0) umma_f16(tmem + (it % NACC) * 112, ad, bd, id, 1);
      __syncwarp();
    }
    if (lane_id() == 0) umma_commit(&bar2);
    mbar_wait(&bar2, 0);
    long long t1 = clock64();
    if (lane_id() == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}

template <typename K>
static void run(K k, const char* what, int bps, int nacc, int astep, int nsm) {
  unsigned long long* dc; CK(cudaMalloc(&dc, 1024 * 8)); CK(cudaMemset(dc, 0, 1024 * 8));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 6144;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<nsm, 128, 200 * 1024>>>(iters, dc);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  }
  std::vector<unsigned long long> c(nsm);
  CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double mx = 0; for (auto v : c) mx = fmax(mx, (double)v);
  printf("%-6s N=112 UMMAs per B slab %2d, accumulators %d, A %s: %.1f cyc/mma (floor 56)\n", what, bps, nacc,
         astep ? "walks 16 B" : "fixed", mx / iters);
  cudaFree(dc);
}

int main() {
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
#define PAIR(B, A, S) run(k_pair<B, A, S>, "pair", B, A, S, nsm)
#define SING(B, A, S) run(k_single<B, A, S>, "single", B, A, S, nsm)
  PAIR(24, 3, 1); PAIR(3, 3, 1); PAIR(3, 3, 0); PAIR(1, 3, 1); PAIR(1, 1, 1); PAIR(1, 1, 0); PAIR(24, 1, 1); PAIR(2, 2, 1);
  SING(24, 3, 1); SING(3, 3, 1); SING(3, 3, 0); SING(1, 3, 1); SING(1, 1, 1); SING(1, 1, 0); SING(24, 1, 1); SING(2, 2, 1);
  printf("PROBE OK\n");
  return 0;
}
