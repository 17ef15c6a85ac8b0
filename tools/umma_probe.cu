// umma_probe.cu — on-device unit tests + microbenchmarks for the tcgen05 building blocks
// the fused kernel relies on (not product code; a development tool).
//  1. plain SS GEMM (fp16 x fp16 -> fp32, K-major SWIZZLE_NONE descriptors)
//  2. "EX" im2col view: A[m][kk] = r[x0 + m + kk] read from an 8x-expanded row (LBO=SBO=128)
//  3. "EY" pair view: A[m][kk] = img[kk][i0 + m] read from two 8-row transposed blocks
//  4. throughput: back-to-back UMMA M=128, N in {112,128,256}, dense vs overlapping A
//  5. TMEM load throughput (32x32b.x16) with 4 and 8 warps
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2107_11627_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace p2s;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct GemmArgs {
  const __half* a_img;  // bytes copied verbatim into smem A region
  int a_bytes;
  const __half* b_img;
  int b_bytes;
  int nsteps;
  uint32_t a_off[8], a_lbo[8], a_sbo[8];  // per K-step A view (offset in bytes into A region)
  uint32_t b_off[8], b_lbo, b_sbo;
  int N;
  float* D;  // [128][N]
};

__global__ void __launch_bounds__(128, 1) k_gemm(GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 65536;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < g.a_bytes; i += 128 * 16)
    *reinterpret_cast<int4*>(sA + i) = *reinterpret_cast<const int4*>((const uint8_t*)g.a_img + i);
  for (int i = threadIdx.x * 16; i < g.b_bytes; i += 128 * 16)
    *reinterpret_cast<int4*>(sB + i) = *reinterpret_cast<const int4*>((const uint8_t*)g.b_img + i);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<256>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    uint32_t id = idesc_f16(128, g.N);
    for (int s = 0; s < g.nsteps; ++s) {
      uint64_t ad = sdesc(smem_u32(sA) + g.a_off[s], g.a_lbo[s], g.a_sbo[s]);
      uint64_t bd = sdesc(smem_u32(sB) + g.b_off[s], g.b_lbo, g.b_sbo);
      umma_f16(tmem, ad, bd, id, s > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  int q = warp_id() & 3;
  for (int c = 0; c < g.N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) g.D[(q * 32 + lane_id()) * g.N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<256>(tmem);
}

// element (row, k) of a K-major SWIZZLE_NONE tile
static size_t kmaj(int row, int k, int lbo, int sbo) {
  return (row % 8) * 16 + (row / 8) * sbo + (k % 8) * 2 + (k / 8) * lbo;
}

static float rnd(unsigned& s) { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; }

static int check(const char* name, const std::vector<float>& D, const std::vector<double>& R) {
  double md = 0, mr = 0;
  for (size_t i = 0; i < D.size(); ++i) { md = fmax(md, fabs(D[i] - R[i])); mr = fmax(mr, fabs(R[i])); }
  bool ok = md <= 1e-3 * fmax(1.0, mr);
  printf("%-28s max|D-R| = %.3e (max|R| %.3f)  %s\n", name, md, mr, ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}

static int run_gemm(const char* name, std::vector<__half>& A, std::vector<__half>& B, GemmArgs g,
                    const std::vector<double>& R) {
  __half *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dD, 128 * g.N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  g.a_img = dA; g.b_img = dB; g.a_bytes = (int)A.size() * 2; g.b_bytes = (int)B.size() * 2; g.D = dD;
  CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
  k_gemm<<<1, 128, 65536 * 2>>>(g);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<float> D(128 * g.N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return check(name, D, R);
}

// --------------------------------------------------------------- throughput
// MODE 0: back-to-back MMAs; MODE 1: + mbarrier try_wait (already complete) every MPS MMAs;
// MODE 2: + tcgen05.commit every MPS MMAs.
template <int N, int OVERLAP, int MODE, int MPS>
__global__ void __launch_bounds__(128, 1) k_tput(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 96 * 1024; i += 128 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tslot;
  if (warp_id() == 0) {
    if (lane_id() == 0) mbar_arrive(&bar2);  // complete phase 0 of bar2
    __syncwarp();
    constexpr uint32_t id = idesc_f16(128, N);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ad[i] = OVERLAP ? sdesc(sa + i * 16 * 5, 128, 128) : sdesc(sa + i * 4096, 128, 256);
      bd[i] = sdesc(sb + i * 8192, 128, 256);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += MPS) {
      if (MODE == 1) mbar_wait(&bar2, 0);
      if (lane_id() == 0) {
#pragma unroll
        for (int j = 0; j < MPS; ++j)
          umma_f16(tmem + (j % 3) * 128, ad[j & 3], bd[(it / MPS) & 3], id, 1);
        if (MODE == 2) umma_commit(&bar);
      }
      __syncwarp();
    }
    if (lane_id() == 0) umma_commit(&bar2);
    mbar_wait(&bar2, 1);
    long long t1 = clock64();
    if (lane_id() == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}

template <int N, int OV, int MODE, int MPS>
static void run_tput(int nsm) {
  unsigned long long* dc; CK(cudaMalloc(&dc, 1024 * 8));
  auto k = k_tput<N, OV, MODE, MPS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 6144;
  for (int grid : {1, nsm}) {
    k<<<grid, 128, 200 * 1024>>>(iters, dc);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<grid, 128, 200 * 1024>>>(iters, dc);
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> c(grid);
    CK(cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost));
    double mx = 0; for (auto v : c) mx = fmax(mx, (double)v);
    double floor_cyc = 128.0 * N / 256.0;
    double tflops = 2.0 * 128 * N * 16 * (double)iters * grid / (ms * 1e-3) / 1e12;
    printf("tput N=%3d A=%-7s mode=%d mps=%d grid=%3d: %.1f cyc/mma (floor %.0f) -> %.0f%% ; %.1f TFLOP/s (%.3f ms)\n",
           N, OV ? "overlap" : "dense", MODE, MPS, grid, mx / iters, floor_cyc, 100.0 * floor_cyc / (mx / iters), tflops, ms);
  }
  cudaFree(dc);
}

__global__ void __launch_bounds__(256, 1) k_tmem_ld(int nwarps, int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t tslot;
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tslot;
  float acc = 0;
  long long t0 = clock64();
  if ((int)warp_id() < nwarps) {
    int q = warp_id() & 3, half = warp_id() >> 2;
    for (int it = 0; it < iters; ++it) {
      for (int c = half * 16; c < 448; c += 16 * (nwarps / 4)) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) acc += v[i];
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}


// ---- 6. interference: UMMA (N=112, M=128, overlapped A) while other warps either stream
// tcgen05.ld from other TMEM columns (mode 1) or spin in mbarrier try_wait (mode 2).
__global__ void __launch_bounds__(384, 1) k_interf(int mode, int iters, unsigned long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar_never;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  for (int i = threadIdx.x * 16; i < 96 * 1024; i += 384 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar_never, 1); done = 0; fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tslot;
  const int w = warp_id();
  if (w == 0 && mode != 3) {
    constexpr uint32_t id = idesc_f16(128, 112);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { ad[i] = sdesc(sa + i * 16 * 5, 128, 128); bd[i] = sdesc(sb + i * 8192, 128, 256); }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 3) {
#pragma unroll
      for (int j = 0; j < 3; ++j) umma_f16_elect(tmem + j * 112, ad[j], bd[(it / 3) & 3], id, 1);
    }
    umma_commit_elect(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) { cyc[blockIdx.x] = (unsigned long long)(t1 - t0); done = 1; }
  } else if ((mode == 1 || mode == 3) && w >= 4) {
    // TMEM readers: 8 warps (2 per lane quadrant) reading columns [384, 512)
    int q = w & 3;
    float acc = 0;
    long long t0 = clock64();
    unsigned long long nld = 0;
    while (!done) {
      for (int c = 384; c < 512; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
        ++nld;
        for (int i = 0; i < 16; ++i) acc += v[i];
      }
    }
    long long t1 = clock64();
    sink[threadIdx.x] = acc;
    if (lane_id() == 0 && blockIdx.x == 0) cyc[1000 + w] = (unsigned long long)((t1 - t0) / (nld ? nld : 1));
  } else if (w == 0 && mode == 3) {
    // no MMA: let the readers run alone for a while
    long long t0 = clock64();
    while (clock64() - t0 < 400000) {}
    if (lane_id() == 0) { cyc[blockIdx.x] = 400000ull * 3 / 6144; done = 1; }
  } else if (mode == 2 && w >= 4) {
    while (!done) { mbar_try_wait(&bar_never, 0); }
  } else if (mode == 4 && w >= 4) {
    // try_wait with an explicit suspend-time hint (ns)
    while (!done) {
      uint32_t ok;
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
          " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(&bar_never)), "r"(0u), "r"(1000000u) : "memory");
    }
  } else if (mode == 5 && w >= 4) {
    // non-blocking test_wait + nanosleep backoff
    while (!done) { if (!mbar_test(&bar_never, 0)) __nanosleep(256); }
  } else if (mode == 6 && w >= 4) {
    // 8 warps streaming 16-B shared stores (what the builders / drains do)
    uint8_t* buf = smem + 160 * 1024 + (w - 4) * 4096;
    int i = 0;
    while (!done) { *reinterpret_cast<int4*>(buf + ((i++ * 512 + lane_id() * 16) & 4095)) = make_int4(i, i, i, i); }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem);
}

static void run_interf(int nsm) {
  unsigned long long* dc; float* sink; CK(cudaMalloc(&dc, 2048 * 8)); CK(cudaMalloc(&sink, 4096 * 4));
  CK(cudaFuncSetAttribute(k_interf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 6144;
  for (int mode = 0; mode < 7; ++mode) {
    k_interf<<<nsm, 384, 200 * 1024>>>(mode, iters, dc, sink);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    k_interf<<<nsm, 384, 200 * 1024>>>(mode, iters, dc, sink);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> c(nsm);
    CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
    double mx = 0; for (auto v : c) mx = fmax(mx, (double)v);
    unsigned long long ldc[16];
    CK(cudaMemcpy(ldc, dc + 1000, 16 * 8, cudaMemcpyDeviceToHost));
    printf("interference mode=%d (%s): %.1f cyc/mma (floor 56); reader cycles per ld16+wait (warp 4): %llu\\n", mode,
           mode == 0 ? "alone" : mode == 1 ? "8 warps tcgen05.ld" : mode == 2 ? "8 warps spin try_wait" : mode == 3 ? "readers alone" :
           mode == 4 ? "8 warps try_wait+suspend hint" : mode == 5 ? "8 warps test_wait+nanosleep" : "8 warps st.shared.v4 stream",
           mx / iters, (mode == 1 || mode == 3) ? ldc[4] : 0ull);
  }
}


// ---- 7. 2-CTA (cluster pair) UMMA throughput: M=256, N=112, A = overlapped E view, B = half per CTA.
// MODE 0: back-to-back; MODE 1: + multicast commit + try_wait (already complete) every MPS UMMAs.
template <int MODE, int MPS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_tput2(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 96 * 1024; i += 128 * 16) *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (warp_id() == 0) tmem_alloc2<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  uint32_t tmem = tslot;
  const bool leader = cluster_ctarank() == 0;
  if (warp_id() == 0 && leader) {
    if (lane_id() == 0) mbar_arrive(&bar2);
    __syncwarp();
    constexpr uint32_t id = idesc_f16(256, 112);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { ad[i] = sdesc(sa + i * 16 * 5, 2624, 128); bd[i] = sdesc(sb + i * 2048, 128, 256); }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += MPS) {
      if (MODE == 1) mbar_wait(&bar2, 0);
#pragma unroll
      for (int j = 0; j < MPS; ++j) umma2_f16_elect(tmem + (j % 3) * 112, ad[j & 3], bd[(it / MPS) & 3], id, 1);
      if (MODE == 1) umma2_commit_elect(&bar);
    }
    umma2_commit_elect(&bar2);
    mbar_wait(&bar2, 1);
    long long t1 = clock64();
    if (lane_id() == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<512>(tmem);
}

template <int MODE, int MPS>
static void run_tput2(int nsm) {
  unsigned long long* dc; CK(cudaMalloc(&dc, 1024 * 8)); CK(cudaMemset(dc, 0, 1024 * 8));
  auto k = k_tput2<MODE, MPS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 6144 / MPS * MPS;
  k<<<nsm, 128, 200 * 1024>>>(iters, dc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  k<<<nsm, 128, 200 * 1024>>>(iters, dc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> c(nsm);
  CK(cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double mx = 0; for (auto v : c) mx = fmax(mx, (double)v);
  printf("2CTA tput M=256 N=112 mode=%d mps=%d: %.1f cyc/mma (floor 56)\n", MODE, MPS, mx / iters);
  cudaFree(dc);
}

int main() {
  int fails = 0;
  unsigned s = 12345;
  const int N = 112;
  // ---- 1. dense GEMM, K = 64 (4 steps); A LBO=128, SBO=1024 ; B LBO=128 SBO=1024
  {
    std::vector<float> a(128 * 64), b(N * 64);
    for (auto& v : a) v = rnd(s);
    for (auto& v : b) v = rnd(s);
    std::vector<__half> A(128 * 64), B(N * 64);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 64; ++k) A[kmaj(m, k, 128, 1024) / 2] = __float2half(a[m * 64 + k]);
    for (int n = 0; n < N; ++n) for (int k = 0; k < 64; ++k) B[kmaj(n, k, 128, 1024) / 2] = __float2half(b[n * 64 + k]);
    std::vector<double> R(128 * N, 0.0);
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < 64; ++k)
      R[m * N + n] += (double)__half2float(A[kmaj(m, k, 128, 1024) / 2]) * __half2float(B[kmaj(n, k, 128, 1024) / 2]);
    GemmArgs g{}; g.nsteps = 4; g.N = N; g.b_lbo = 128; g.b_sbo = 1024;
    for (int t = 0; t < 4; ++t) { g.a_off[t] = t * 256; g.a_lbo[t] = 128; g.a_sbo[t] = 1024; g.b_off[t] = t * 256; }
    fails += run_gemm("dense K-major GEMM", A, B, g, R);
  }
  // ---- 2. EX view: EX[i][j] = r[i + j], A[m][kk] = r[x0 + m + kk]
  {
    const int NP = 200, x0 = 13;
    std::vector<float> r(NP + 8), b(N * 16);
    for (auto& v : r) v = rnd(s);
    for (auto& v : b) v = rnd(s);
    std::vector<__half> A(NP * 8), B(N * 16);
    for (int i = 0; i < NP; ++i) for (int j = 0; j < 8; ++j) A[i * 8 + j] = __float2half(r[i + j]);
    for (int n = 0; n < N; ++n) for (int k = 0; k < 16; ++k) B[kmaj(n, k, 128, 256) / 2] = __float2half(b[n * 16 + k]);
    std::vector<double> R(128 * N, 0.0);
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < 16; ++k)
      R[m * N + n] += (double)__half2float(__float2half(r[x0 + m + k])) * __half2float(B[kmaj(n, k, 128, 256) / 2]);
    GemmArgs g{}; g.nsteps = 1; g.N = N; g.b_lbo = 128; g.b_sbo = 256;
    g.a_off[0] = x0 * 16; g.a_lbo[0] = 128; g.a_sbo[0] = 128; g.b_off[0] = 0;
    fails += run_gemm("EX overlapped view", A, B, g, R);
  }
  // ---- 3. EY pair: EYb[i][j] = img[8b + j][i]; A[m][kk] = img[kk][i0 + m]; plus V8 pair LBO=16
  {
    const int NP = 200, i0 = 21;
    std::vector<float> img(16 * NP), b(N * 16);
    for (auto& v : img) v = rnd(s);
    for (auto& v : b) v = rnd(s);
    std::vector<__half> A(2 * NP * 8), B(N * 16);
    for (int blk = 0; blk < 2; ++blk) for (int i = 0; i < NP; ++i) for (int j = 0; j < 8; ++j)
      A[(blk * NP + i) * 8 + j] = __float2half(img[(8 * blk + j) * NP + i]);
    for (int n = 0; n < N; ++n) for (int k = 0; k < 16; ++k) B[kmaj(n, k, 128, 256) / 2] = __float2half(b[n * 16 + k]);
    std::vector<double> R(128 * N, 0.0), R2(128 * N, 0.0);
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < 16; ++k) {
      double bb = __half2float(B[kmaj(n, k, 128, 256) / 2]);
      R[m * N + n] += (double)__half2float(__float2half(img[k * NP + i0 + m])) * bb;
      // V8 pair: core h = column i0+m+h, rows j  => A[m][kk] = img[kk%8][i0 + m + kk/8]
      R2[m * N + n] += (double)__half2float(__float2half(img[(k % 8) * NP + i0 + m + k / 8])) * bb;
    }
    GemmArgs g{}; g.nsteps = 1; g.N = N; g.b_lbo = 128; g.b_sbo = 256;
    g.a_off[0] = i0 * 16; g.a_lbo[0] = NP * 16; g.a_sbo[0] = 128; g.b_off[0] = 0;
    fails += run_gemm("EY pair view (LBO=block)", A, B, g, R);
    g.a_lbo[0] = 16;
    fails += run_gemm("EY V8 view (LBO=16)", A, B, g, R2);
  }
  // ---- 4. throughput
  {
    int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    run_tput<112, 0, 0, 3>(nsm); run_tput<112, 1, 0, 3>(nsm);
    run_tput<128, 0, 0, 3>(nsm); run_tput<128, 1, 0, 3>(nsm);
    run_tput<256, 0, 0, 2>(nsm); run_tput<256, 1, 0, 2>(nsm);
    run_tput<112, 1, 1, 3>(nsm); run_tput<112, 1, 2, 3>(nsm);
    run_tput<112, 1, 1, 6>(nsm); run_tput<112, 1, 2, 6>(nsm);
    run_tput<208, 0, 0, 2>(nsm); run_tput<64, 0, 0, 4>(nsm);
  }
  { int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0)); run_interf(nsm);
    run_tput2<0, 24>(nsm); run_tput2<1, 24>(nsm); run_tput2<1, 12>(nsm); run_tput2<1, 48>(nsm); }
  // ---- 5. TMEM load throughput
  {
    unsigned long long* dc; float* sink; CK(cudaMalloc(&dc, 8)); CK(cudaMalloc(&sink, 1024 * 4));
    for (int nw : {4, 8}) {
      const int iters = 200;
      k_tmem_ld<<<1, 256>>>(nw, iters, dc, sink);
      CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
      unsigned long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
      double bytes = (double)iters * 128 * 448 * 4;
      printf("tmem ld32x32b.x16 with %d warps: %.0f cycles for %.0f KB -> %.1f B/cyc\n", nw, (double)c, bytes / 1024, bytes / c);
    }
  }
  printf("%s (%d failures)\n", fails ? "PROBE FAILED" : "PROBE OK", fails);
  return fails ? 1 : 0;
}
