// p2s_kernels.cuh — device side of the P2S hot path (sm_100a).
//
//  k_fused_p2s  steps a0+a1+a2: per 128-pixel tile (one image row segment), the P2S MLP
//                and the K invariant convolutions combined per output
//               pixel (Eq. 5) on tcgen05 tensor cores, fp16 operands,
//               fp32 accumulation in TMEM; beta and the K x C convolution results never
//               leave the SM; writes J [B][C][H][W] fp32.
//  k_tilt_warp  step a3: backward bilinear warp with clamp-to-edge.
//
// Layouts:
//  * UMMA operands use the SWIZZLE_NONE K-major canonical layout: element (row, k) at
//    (row%8)*16 + (row/8)*SBO + (k%8)*2 + (k/8)*LBO.
//  * B operands (weights, basis) are pre-packed on the host into 16-K "slabs"
//    (LBO = 128, SBO = 256 -> rows*32 bytes) and streamed by the bulk-copy engine into a
//    ring of multi-slab stages.
//  * The convolution A operand (im2col, one input channel) is never materialised per
//    K-step: an 8x-expanded view of the image ("EY" blocks: 8 consecutive rows of one
//    column per 16-byte entry; "EX" rows: 8 consecutive columns of one row) is built once
//    per tile, and each K-step addresses it with an overlapping descriptor (SBO = 16 B per
//    pixel row, LBO = block stride / 128 B / 16 B). See plan_conv() in p2s_host.cu.
#pragma once
#include "sm100.cuh"

namespace p2s {

constexpr int kTileM = 128;          // pixels per tile (UMMA M)
constexpr int kThreads = 320;        // 10 warps
constexpr int kWarpProducer = 0;     // bulk-copy producer (lane 0)
constexpr int kWarpMma = 1;          // UMMA issuer (lane 0) + TMEM owner
constexpr int kWarpBuild0 = 2;       // warps 2..5: A1 (Zernike tile) and E (im2col views)
constexpr int kWarpEpi0 = 6;         // warps 6..9: TMEM drains, MLP activations, J epilogue
constexpr int kBuildThreads = 128;
constexpr int kEpiThreads = 128;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kBetaCol = 384;   // beta (L3 accumulator) lives in columns [384, 384+Nk)
constexpr int kMaxStages = 128;      // per-tile stage list capacity
constexpr int kMaxConvSteps = 512;
constexpr int kMaxEy = 16, kMaxEx = 4;

// One ring stage = nslabs consecutive 16-K slabs of one layer, contiguous in the stream.
struct StageDesc {
  uint32_t src_off;   // byte offset in the packed stream
  uint32_t bytes;     // nslabs * slab_bytes
  uint32_t layer;     // 0,1,2 = MLP layers, 3 = convolution
  uint32_t first;     // index of the first slab (K-step) within its layer
};

struct FusedParams {
  const float* image;    // [B][C][H][W]
  const float* zernike;  // [B][n_in][H][W]
  float* J;              // [B][C][H][W] (mode 0)
  float* beta_out;       // [B][K][H][W] (mode 1)
  int B, C, H, W, n_in;
  int nstrips, ntiles, mode;  // mode 0: MLP + conv -> J ; mode 1: MLP only -> beta
  const uint8_t* stream;
  const StageDesc* stages;
  int nst_l[4];               // number of stages of each layer per tile
  int nstages;                // nst_l[0]+...+nst_l[3]
  const uint2* conv_steps;    // per conv K-step: (A byte offset in a channel's E region, LBO)
  int nconv;
  const float *b1, *b2, *b3, *svec;  // padded biases; svec[k] = sum of taps of phi_k
  int K, Nk, K1, N1, N2;
  int r;
  int n_ey, n_ex, npos_y, npos_x;
  int ey_a0[kMaxEy], ex_a[kMaxEx];
  int chan_bytes;             // E region bytes per channel
  int stage_bytes, nring;
  int off_ring, off_a1, off_a2, off_e, off_tab, off_bar, smem_bytes;
  int a1_sbo, a2_sbo;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// barrier slots in shared memory
enum Bar {
  BAR_A1_FULL = 0, BAR_A1_EMPTY, BAR_E_FULL, BAR_E_EMPTY, BAR_MLP_DONE, BAR_A2_FULL,
  BAR_ACC_FULL, BAR_TMEM_FREE, BAR_RING = 8  // then ring_full[n], ring_empty[n]
};

__device__ __forceinline__ void tile_coords(const FusedParams& p, int t, int& b, int& y, int& x0) {
  const int per_b = p.nstrips * p.H;
  b = t / per_b;
  const int rem = t - b * per_b;
  const int s = rem / p.H;
  y = rem - s * p.H;
  x0 = s * kTileM;
}

__global__ void __launch_bounds__(kThreads, 1) k_fused_p2s(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* ring_full = bars + BAR_RING;
  uint64_t* ring_empty = bars + BAR_RING + p.nring;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + BAR_RING + 2 * p.nring);
  uint8_t* ring = smem + p.off_ring;
  uint8_t* sA1 = smem + p.off_a1;
  uint8_t* sA2 = smem + p.off_a2;
  uint8_t* sE = smem + p.off_e;
  StageDesc* sStages = reinterpret_cast<StageDesc*>(smem + p.off_tab);
  uint2* sSteps = reinterpret_cast<uint2*>(smem + p.off_tab + kMaxStages * sizeof(StageDesc));

  const int warp = warp_id();
  const int lane = lane_id();

  // per-CTA contiguous range of tiles
  const int t_begin = (int)(((long long)blockIdx.x * p.ntiles) / gridDim.x);
  const int t_end = (int)(((long long)(blockIdx.x + 1) * p.ntiles) / gridDim.x);

  // ---- setup
  for (int i = threadIdx.x; i < p.nstages; i += kThreads) sStages[i] = p.stages[i];
  for (int i = threadIdx.x; i < p.nconv; i += kThreads) sSteps[i] = p.conv_steps[i];
  if (threadIdx.x == 0) {
    mbar_init(&bars[BAR_A1_FULL], kBuildThreads / 32);
    mbar_init(&bars[BAR_A1_EMPTY], 1);
    mbar_init(&bars[BAR_E_FULL], kBuildThreads / 32);
    mbar_init(&bars[BAR_E_EMPTY], 1);
    mbar_init(&bars[BAR_MLP_DONE], 1);
    mbar_init(&bars[BAR_A2_FULL], kEpiThreads / 32);
    mbar_init(&bars[BAR_ACC_FULL], 1);
    mbar_init(&bars[BAR_TMEM_FREE], kEpiThreads / 32);
    for (int i = 0; i < p.nring; ++i) { mbar_init(&ring_full[i], 1); mbar_init(&ring_empty[i], 1); }
    fence_mbar_init();
  }
  if (warp == kWarpMma) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nst_tile = p.mode == 0 ? p.nstages : p.nst_l[0] + p.nst_l[1] + p.nst_l[2];

  if (warp == kWarpProducer) {
    // ================= producer: stream weight/basis slabs into the ring =================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = t_begin; t < t_end; ++t) {
        for (int g = 0; g < nst_tile; ++g) {
          const StageDesc sd = sStages[g];
          mbar_wait(&ring_empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&ring_full[s], sd.bytes);
          bulk_g2s(ring + (size_t)s * p.stage_bytes, p.stream + sd.src_off, sd.bytes, &ring_full[s]);
          if (++s == p.nring) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ================= UMMA issuer (single thread) =================
    if (lane == 0) {
      const uint32_t ring_s = smem_u32(ring), a1_s = smem_u32(sA1), a2_s = smem_u32(sA2),
                     e_s = smem_u32(sE);
      const uint32_t id_l[4] = {idesc_f16(128, p.N1), idesc_f16(128, p.N2), idesc_f16(128, p.Nk),
                                idesc_f16(128, p.Nk)};
      const uint32_t slab_l[4] = {(uint32_t)p.N1 * 32u, (uint32_t)p.N2 * 32u, (uint32_t)p.Nk * 32u,
                                  (uint32_t)p.Nk * 32u};
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = t_begin; t < t_end; ++t, ++it) {
        int g = 0;
        for (int layer = 0; layer < (p.mode == 0 ? 4 : 3); ++layer) {
          // layer entry dependencies
          if (layer == 0) {
            mbar_wait(&bars[BAR_A1_FULL], it & 1);
            mbar_wait(&bars[BAR_TMEM_FREE], (it & 1) ^ 1);
          } else if (layer == 1) {
            mbar_wait(&bars[BAR_A2_FULL], 0);
          } else if (layer == 2) {
            mbar_wait(&bars[BAR_A2_FULL], 1);
          } else {
            mbar_wait(&bars[BAR_E_FULL], it & 1);
          }
          tc_fence_after();
          const uint32_t dcol = layer == 2 ? kBetaCol : 0u;
          for (int gl = 0; gl < p.nst_l[layer]; ++gl, ++g) {
            const StageDesc sd = sStages[g];
            mbar_wait(&ring_full[s], ph);
            tc_fence_after();
            const uint32_t nsl = sd.bytes / slab_l[layer];
            const uint32_t bbase = ring_s + (uint32_t)s * p.stage_bytes;
            for (uint32_t j = 0; j < nsl; ++j) {
              const uint32_t ks = sd.first + j;
              const uint64_t bd = sdesc(bbase + j * slab_l[layer], 128, 256);
              if (layer < 3) {
                const uint64_t ad = layer == 0 ? sdesc(a1_s + ks * 256, 128, p.a1_sbo)
                                               : sdesc(a2_s + ks * 256, 128, p.a2_sbo);
                umma_f16(tmem + dcol, ad, bd, id_l[layer], ks > 0);
              } else {
                const uint2 st = sSteps[ks];
                for (int c = 0; c < p.C; ++c) {
                  const uint64_t ad = sdesc(e_s + c * p.chan_bytes + st.x, st.y, 128);
                  umma_f16(tmem + c * p.Nk, ad, bd, id_l[3], ks > 0);
                }
              }
            }
            umma_commit(&ring_empty[s]);
            if (++s == p.nring) { s = 0; ph ^= 1; }
          }
          if (layer == 0) umma_commit(&bars[BAR_A1_EMPTY]);
          if (layer == 0 || layer == 1) umma_commit(&bars[BAR_MLP_DONE]);
          if (layer == 2 && p.mode == 1) umma_commit(&bars[BAR_ACC_FULL]);
          if (layer == 3) {
            umma_commit(&bars[BAR_E_EMPTY]);
            umma_commit(&bars[BAR_ACC_FULL]);
          }
        }
      }
    }
  } else if (warp >= kWarpBuild0 && warp < kWarpBuild0 + kBuildThreads / 32) {
    // ================= builders: A1 (Zernike tile, fp16) and E views (fp16, centred) =====
    const int tid = threadIdx.x - kWarpBuild0 * 32;
    const size_t HW = (size_t)p.H * p.W;
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      int b, y, x0;
      tile_coords(p, t, b, y, x0);
      // --- A1: row m = pixel x0+m, k = Zernike index (zero-padded to K1)
      mbar_wait(&bars[BAR_A1_EMPTY], (it & 1) ^ 1);
      {
        const int m = tid;
        const int x = min(x0 + m, p.W - 1);
        const float* zp = p.zernike + (size_t)b * p.n_in * HW + (size_t)y * p.W + x;
        uint8_t* dst = sA1 + (m & 7) * 16 + (m >> 3) * p.a1_sbo;
        for (int k0 = 0; k0 < p.K1; k0 += 8) {
          float v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = (k0 + i < p.n_in) ? __ldg(zp + (size_t)(k0 + i) * HW) : 0.f;
          uint4 q = make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                               pack_half2(v[6], v[7]));
          *reinterpret_cast<uint4*>(dst + (k0 >> 3) * 128) = q;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[BAR_A1_FULL]);
      if (p.mode != 0) continue;
      // --- E views for every channel
      mbar_wait(&bars[BAR_E_EMPTY], (it & 1) ^ 1);
      for (int c = 0; c < p.C; ++c) {
        const float* img = p.image + ((size_t)b * p.C + c) * HW;
        uint8_t* Ec = sE + (size_t)c * p.chan_bytes;
        for (int blk = 0; blk < p.n_ey; ++blk) {
          const float* rows[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            rows[j] = img + (size_t)clampi(y - p.r + p.ey_a0[blk] + j, 0, p.H - 1) * p.W;
          uint8_t* dst = Ec + (size_t)blk * p.npos_y * 16;
          for (int i = tid; i < p.npos_y; i += kBuildThreads) {
            const int col = clampi(x0 - p.r + i, 0, p.W - 1);
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldg(rows[j] + col) - 0.5f;
            *reinterpret_cast<uint4*>(dst + i * 16) =
                make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                           pack_half2(v[6], v[7]));
          }
        }
        for (int e = 0; e < p.n_ex; ++e) {
          const float* row = img + (size_t)clampi(y - p.r + p.ex_a[e], 0, p.H - 1) * p.W;
          uint8_t* dst = Ec + (size_t)p.n_ey * p.npos_y * 16 + (size_t)e * p.npos_x * 16;
          for (int i = tid; i < p.npos_x; i += kBuildThreads) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldg(row + clampi(x0 - p.r + i + j, 0, p.W - 1)) - 0.5f;
            *reinterpret_cast<uint4*>(dst + i * 16) =
                make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                           pack_half2(v[6], v[7]));
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[BAR_E_FULL]);
    }
  } else if (warp >= kWarpEpi0) {
    // ================= epilogue: MLP activations, beta, J =================
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;            // pixel (row of every accumulator)
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const size_t HW = (size_t)p.H * p.W;
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      int b, y, x0;
      tile_coords(p, t, b, y, x0);
      // hidden layers: D (cols [0,N)) -> +bias, ReLU -> fp16 -> A2 (K-major, k = column)
      for (int layer = 0; layer < 2; ++layer) {
        const int N = layer == 0 ? p.N1 : p.N2;
        const float* bias = layer == 0 ? p.b1 : p.b2;
        mbar_wait(&bars[BAR_MLP_DONE], layer);
        tc_fence_after();
        uint8_t* dst = sA2 + (m & 7) * 16 + (m >> 3) * p.a2_sbo;
        for (int c0 = 0; c0 < N; c0 += 16) {
          float v[16];
          tmem_ld16(tl + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + __ldg(bias + c0 + i), 0.f);
          *reinterpret_cast<uint4*>(dst + (c0 >> 3) * 128) =
              make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                         pack_half2(v[6], v[7]));
          *reinterpret_cast<uint4*>(dst + ((c0 >> 3) + 1) * 128) =
              make_uint4(pack_half2(v[8], v[9]), pack_half2(v[10], v[11]), pack_half2(v[12], v[13]),
                         pack_half2(v[14], v[15]));
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[BAR_A2_FULL]);
      }
      mbar_wait(&bars[BAR_ACC_FULL], it & 1);
      tc_fence_after();
      const int x = x0 + m;
      if (p.mode == 1) {
        for (int k0 = 0; k0 < p.Nk; k0 += 16) {
          float bv[16];
          tmem_ld16(tl + kBetaCol + k0, bv);
          tmem_ld_wait();
          if (x < p.W)
            for (int i = 0; i < 16 && k0 + i < p.K; ++i)
              p.beta_out[((size_t)b * p.K + k0 + i) * HW + (size_t)y * p.W + x] = bv[i] + __ldg(p.b3 + k0 + i);
        }
      } else {
        float jc[3] = {0.f, 0.f, 0.f};
        float bs = 0.f;
        for (int k0 = 0; k0 < p.Nk; k0 += 16) {
          float bv[16], av[3][16];
          tmem_ld16(tl + kBetaCol + k0, bv);
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < p.C) tmem_ld16(tl + c * p.Nk + k0, av[c]);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float be = bv[i] + __ldg(p.b3 + k0 + i);
            bs = fmaf(be, __ldg(p.svec + k0 + i), bs);
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c < p.C) jc[c] = fmaf(be, av[c][i], jc[c]);
          }
        }
        if (x < p.W)
          for (int c = 0; c < p.C; ++c)
            p.J[((size_t)b * p.C + c) * HW + (size_t)y * p.W + x] = fmaf(0.5f, bs, jc[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[BAR_TMEM_FREE]);
    }
  }
  // ---- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpMma) tmem_dealloc<kTmemCols>(tmem);
}

// Step a3: out(y,x) = bilinear J at (y - t1, x - t0), clamp-to-edge; all channels per thread.
__global__ void __launch_bounds__(256) k_tilt_warp(const float* __restrict__ J, const float* __restrict__ tilt,
                                                   float* __restrict__ out, int B, int C, int H, int W) {
  const size_t HW = (size_t)H * W;
  const size_t n = (size_t)B * HW;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / HW, pix = i - b * HW;
    const int y = (int)(pix / W), x = (int)(pix - (size_t)y * W);
    float tx = 0.f, ty = 0.f;
    if (tilt) {
      tx = __ldg(tilt + (b * 2 + 0) * HW + pix);
      ty = __ldg(tilt + (b * 2 + 1) * HW + pix);
    }
    const float sy = fminf(fmaxf((float)y - ty, -1.f), (float)H);
    const float sx = fminf(fmaxf((float)x - tx, -1.f), (float)W);
    const float fy0 = floorf(sy), fx0 = floorf(sx);
    const float fy = sy - fy0, fx = sx - fx0;
    const int y0 = (int)fy0, x0 = (int)fx0;
    const int ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
    const int xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
    const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx, w10 = fy * (1.f - fx), w11 = fy * fx;
    for (int c = 0; c < C; ++c) {
      const float* Jc = J + (b * C + c) * HW;
      const float v = w00 * __ldg(Jc + (size_t)ya * W + xa) + w01 * __ldg(Jc + (size_t)ya * W + xb) +
                      w10 * __ldg(Jc + (size_t)yb * W + xa) + w11 * __ldg(Jc + (size_t)yb * W + xb);
      out[(b * C + c) * HW + pix] = v;
    }
  }
}

}  // namespace p2s
