// tmem_a_probe.cu — on-device check of the tcgen05 A-from-TMEM form (dev tool, not product):
//   D[128 x N] = A[128 x K] * B[N x K]^T with A written to TMEM by tcgen05.st (lane = row m,
//   column c = fp16 pair (k = 2c, 2c+1) of one 16-wide K-step block of 8 columns), B in shared
//   memory (SWIZZLE_NONE K-major), mixed K-steps (A from TMEM for some, shared memory for others),
//   and the throughput of back-to-back UMMAs with A in TMEM vs shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace p2s;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void umma_tA(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
      "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_tA_elect(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n .reg .pred e, p;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
      "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

constexpr int KS = 4;  // K-steps (K = 64)

// A [128][64] fp16 row-major, B [N][64] fp16 row-major; tmask bit s: K-step s reads A from TMEM
__global__ void __launch_bounds__(128, 1) k_check(const __half* A, const __half* B, int N, int tmask, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;           // [128][64] K-major canonical: (m%8)*16 + (m/8)*1024 + (k%8)*2 + (k/8)*128
  uint8_t* sB = smem + 16384;   // [N][64]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int m = 0; m < 128; m += 1)
    for (int k = t; k < 64; k += 128) {}
  // canonical layouts (kd = 64 -> SBO = 8 rows * 64 * 2 = 1024, LBO = 128)
  for (int e = t; e < 128 * 64; e += 128) {
    const int m = e / 64, k = e % 64;
    *reinterpret_cast<__half*>(sA + (m % 8) * 16 + (m / 8) * 1024 + (k % 8) * 2 + (k / 8) * 128) = A[e];
  }
  for (int e = t; e < N * 64; e += 128) {
    const int n = e / 64, k = e % 64;
    *reinterpret_cast<__half*>(sB + (n % 8) * 16 + (n / 8) * 1024 + (k % 8) * 2 + (k / 8) * 128) = B[e];
  }
  fence_proxy_async_smem();
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int q = warp_id() & 3, m = t;  // 128 threads: thread m owns lane m
  const uint32_t a_col = 256;
  // A -> TMEM: K-step s occupies columns a_col + 8 s .. + 7, column c = pair (2c, 2c+1)
  for (int s = 0; s < KS; ++s) {
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) {
      __half2 h = __halves2half2(A[m * 64 + s * 16 + 2 * c], A[m * 64 + s * 16 + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st8(tmem + ((uint32_t)(q * 32) << 16) + a_col + 8 * s, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint32_t id = idesc_f16(128, N);
    for (int s = 0; s < KS; ++s) {
      const uint64_t bd = sdesc(smem_u32(sB) + s * 256, 128, 1024);
      if ((tmask >> s) & 1) umma_tA(tmem, tmem + a_col + 8 * s, bd, id, s > 0);
      else umma_f16(tmem, sdesc(smem_u32(sA) + s * 256, 128, 1024), bd, id, s > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) D[m * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}

// throughput: n back-to-back UMMAs M = 128, N, K = 16, A from TMEM (mode 1) or smem (mode 0)
__global__ void __launch_bounds__(128, 1) k_tput(int N, int mode, int n, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp_id() == 0) {  // whole warp, uniform operands, elected lane issues (as the product kernels)
    const uint32_t id = idesc_f16(128, N);
    const uint32_t sb = smem_u32(smem);
    const uint64_t a_hi = ((uint64_t)((1024u >> 4)) << 32) | (1ull << 46), b_hi = ((uint64_t)((4096u >> 4)) << 32) | (1ull << 46);
    const long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
      const uint64_t bd = b_hi | ((uint64_t)(128u >> 4) << 16) | (((sb + 65536u + (uint32_t)(i & 3) * 256u) >> 4) & 0x3FFFu);
      if (mode) umma_tA_elect(tmem, tmem + 256 + 8 * (i & 7), bd, id, 1);
      else umma_f16_elect(tmem, a_hi | ((uint64_t)(128u >> 4) << 16) | (((sb + (uint32_t)(i & 3) * 256u) >> 4) & 0x3FFFu), bd, id, 1);
    }
    umma_commit_elect(&bar);
    mbar_wait(&bar, 0);
    if (lane_id() == 0) cyc[0] = clock64() - t0;
  }
  __syncthreads();
  tc_fence_after();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}

int main() {
  const int N = 208;
  std::vector<__half> A(128 * 64), B(N * 64);
  std::vector<float> Af(128 * 64), Bf(N * 64);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) { float v = (rand() % 2001 - 1000) / 1000.f; A[i] = __float2half(v); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * 64; ++i) { float v = (rand() % 2001 - 1000) / 1000.f; B[i] = __float2half(v); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
  CK(cudaFuncSetAttribute(k_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  std::vector<float> D(128 * N);
  for (int tmask : {0x0, 0xF, 0x5, 0xA, 0x1, 0x8}) {
    CK(cudaMemset(dD, 0, 128 * N * 4));
    k_check<<<1, 128, 100000>>>(dA, dB, N, tmask, dD);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < 64; ++k) r += (double)Af[m * 64 + k] * Bf[n * 64 + k];
        err = fmax(err, fabs(r - D[m * N + n]));
      }
    printf("A-from-TMEM check tmask=0x%x: max |D - ref| = %.3e %s\n", tmask, err, err < 1e-3 ? "OK" : "FAIL");
  }
  long long* dc;
  CK(cudaMalloc(&dc, 8));
  for (int n : {48, 112, 208, 256})
    for (int mode : {0, 1}) {
      long long c = 0;
      for (int rep = 0; rep < 3; ++rep) {
        k_tput<<<1, 128, 200000>>>(n, mode, 512, dc);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
      printf("throughput N=%d A from %s: %.1f cycles per UMMA (M=128, K=16; floor %.1f)\n", n, mode ? "TMEM" : "smem",
             c / 512.0, 128.0 * n * 16 / 4096.0);
    }
  return 0;
}
