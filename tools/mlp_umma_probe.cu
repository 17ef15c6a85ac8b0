// mlp_umma_probe.cu — pair (cta_group::2, M = 256) UMMA throughput for the fused kernel's MLP
// chunks (dev tool, not product code): A = a K-major SWIZZLE_NONE activation tile ([128][208] fp16
// per CTA, SBO = 3328 B), B = per-K-step slab halves ([N/2][16], LBO 128, SBO 256), N in
// {48, 80, 112, 128, 208, 256}; cycles per UMMA with the SMs otherwise idle, with 8 warps per CTA
// reading TMEM (tcgen05.ld of other columns, as the drains do) and with 8 warps storing to shared
// memory (as the drains' A-operand writes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace p2s;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// mode 0: idle; 1: 8 warps tcgen05.ld columns [256, 512); 2: 8 warps st.shared into a scratch area;
// 3/4: warp 1 streams global -> shared bulk copies into a scratch area while the UMMAs run (3: 1.8 KB
// copies, the fused kernel's per-slab TMA boxes; 4: 19.7 KB copies, one per ring stage)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(288, 1)
    k_mlp(int N, int n, int mode, unsigned long long* cyc, const uint8_t* src) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  for (int i = threadIdx.x * 16; i < 200 * 1024; i += 288 * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0x3c003c00, 0x3c003c00, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool leader = cluster_ctarank() == 0;
  const int warp = warp_id();
  if (warp == 0) {
    if (leader) {
      const uint32_t id = idesc_f16(256, (uint32_t)N);
      const uint32_t a_lo = (smem_u32(smem) >> 4) | ((128u >> 4) << 16);
      const uint32_t b_lo = (smem_u32(smem + 64 * 1024) >> 4) | ((128u >> 4) << 16);
      const uint64_t hi_a = ((uint64_t)((3328u >> 4) | (1u << 14))) << 32, hi_b = ((uint64_t)((256u >> 4) | (1u << 14))) << 32;
      const uint32_t bstep = (uint32_t)N * 16u >> 4;  // one CTA's half slab: N/2 rows x 32 B
      const long long t0 = clock64();
#pragma unroll 2
      for (int i = 0; i < n; ++i)
        umma2_f16_elect(tmem, hi_a | (a_lo + (uint32_t)(i % 13) * 16u), hi_b | (b_lo + (uint32_t)(i % 13) * bstep), id,
                        i > 0);
      umma2_commit_elect(&bar);
      mbar_wait(&bar, 0);
      if (lane_id() == 0) cyc[0] = clock64() - t0;
    } else {
      mbar_wait(&bar, 0);
    }
    __syncwarp();
    if (lane_id() == 0) done = 1;
  } else if (warp == 1 && mode >= 3) {
    // bulk copies, up to 3 in flight (a 3-stage ring), into [160 KB, 200 KB)
    __shared__ uint64_t cb[3];
    if (lane_id() == 0) {
      for (int i = 0; i < 3; ++i) mbar_init(&cb[i], 1);
      fence_mbar_init();
      const uint32_t bytes = mode == 3 ? 1792u : 19712u;
      uint32_t ph[3] = {0, 0, 0};
      int it = 0;
      while (!done && it < 200000) {
        const int s = it % 3;
        if (it >= 3) { mbar_wait(&cb[s], ph[s]); ph[s] ^= 1u; }
        mbar_arrive_expect_tx(&cb[s], bytes);
        bulk_g2s(smem + 160 * 1024 + (mode == 3 ? s * 2048 : 0), src + (size_t)(it % 64) * 32768, bytes, &cb[s]);
        ++it;
      }
      for (int s = 0; s < 3 && it >= 3; ++s) { mbar_wait(&cb[(it + s) % 3], ph[(it + s) % 3]); }
      cyc[1] = it;
    }
    __syncwarp();
  } else if (warp >= 1 && mode != 0 && mode < 3) {
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t acc = 0;
    int it = 0;
    while (!done && it < 100000) {
      if (mode == 1) {
        float v[16];
        tmem_ld16(tq + 256u + (uint32_t)((it & 7) * 16), v);
        tmem_ld_wait();
        acc += __float_as_uint(v[0]) ^ __float_as_uint(v[15]);
      } else {
        uint4* p = reinterpret_cast<uint4*>(smem + 160 * 1024 + ((threadIdx.x * 16 + it * 4608) & 32767));
        *p = make_uint4(acc, it, 1, 2);
        acc += 3;
      }
      ++it;
    }
    if (acc == 12345u) cyc[1] = acc;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc2<512>(tmem);
}

int main() {
  unsigned long long* d;
  CK(cudaMalloc(&d, 16));
  uint8_t* src;
  CK(cudaMalloc(&src, 64 * 32768 + 65536));
  CK(cudaMemset(src, 0, 64 * 32768 + 65536));
  CK(cudaFuncSetAttribute(k_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const char* names[] = {"idle", "8 warps tcgen05.ld", "8 warps st.shared", "bulk 1.8 KB copies", "bulk 19.7 KB copies"};
  for (int mode = 0; mode < 5; ++mode)
    for (int N : {48, 80, 112, 128, 208, 256}) {
      unsigned long long c = 0;
      for (int rep = 0; rep < 3; ++rep) {
        k_mlp<<<2, 288, 200 * 1024>>>(N, 390, mode, d, src);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost));
      printf("%-20s N=%3d: %6.1f cycles per pair UMMA (M=256, K=16; floor %5.1f)\n", names[mode], N, c / 390.0,
             256.0 * N * 16 / 8192.0);
    }
  return 0;
}
