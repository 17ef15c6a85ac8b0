// launch_probe.cu — GPU-side cost of launching a kernel shaped like k_fused_p2s (dev tool): back-to-back
// launches of empty kernels, CUDA events around each, for: plain 148 x 448 threads; + clusters of 2;
// + 227 KB dynamic shared memory; + TMEM alloc/dealloc (cta_group::2); + a 2 KB __grid_constant__
// parameter block.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace p2s;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1;} } while (0)

struct Big { unsigned char b[2048]; };
__global__ void __launch_bounds__(448) k_plain(int* o) { if (o && threadIdx.x == 9999) o[0] = 1; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(448) k_cluster(int* o) { if (o && threadIdx.x == 9999) o[0] = 1; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(448) k_tmem(int* o) {
  __shared__ uint32_t slot;
  if (warp_id() == 2) tmem_alloc2<512>(&slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t t = slot;
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp_id() == 2) tmem_dealloc2<512>(t);
  if (o && threadIdx.x == 9999) o[0] = 1;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(448) k_big(const __grid_constant__ Big b, int* o) {
  if (o && threadIdx.x == 9999) o[0] = b.b[threadIdx.x & 2047];
}

template <typename F>
float timeit(F f, int n) {
  cudaEvent_t a[64], b[64];
  for (int i = 0; i < n; ++i) { cudaEventCreate(&a[i]); cudaEventCreate(&b[i]); }
  for (int i = 0; i < 20; ++i) f();
  for (int i = 0; i < n; ++i) { cudaEventRecord(a[i]); f(); cudaEventRecord(b[i]); }
  cudaDeviceSynchronize();
  float tot = 0;
  for (int i = 0; i < n; ++i) { float ms; cudaEventElapsedTime(&ms, a[i], b[i]); tot += ms; }
  return tot / n * 1e3f;
}

int main() {
  const int smem = 232448 - 2048;
  CK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  Big big{};
  printf("plain 148x448:                     %6.2f us\n", timeit([&] { k_plain<<<148, 448>>>(nullptr); }, 50));
  printf("clusters of 2:                     %6.2f us\n", timeit([&] { k_cluster<<<148, 448>>>(nullptr); }, 50));
  printf("clusters + 227 KB smem:            %6.2f us\n", timeit([&] { k_cluster<<<148, 448, smem>>>(nullptr); }, 50));
  printf("clusters + smem + TMEM alloc:      %6.2f us\n", timeit([&] { k_tmem<<<148, 448, smem>>>(nullptr); }, 50));
  printf("clusters + smem + 2 KB params:     %6.2f us\n", timeit([&] { k_big<<<148, 448, smem>>>(big, nullptr); }, 50));
  return 0;
}
