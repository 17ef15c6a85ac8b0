// p2s_mlp_backward.cuh — dL/dz through the P2S MLP: the adjoint of step a1 (PAPER.md:280-283
// "three fully connected layers", reading A11: ReLU after layers 1-2, linear output; the
// simulator "as a differentiable module").
//
// Per pixel, for z in R^n_in and g3 = dL/dbeta in R^K:
//     pre1 = W1 z + b1,  a1 = ReLU(pre1),  pre2 = W2 a1 + b2
//     g2 = (W3^T g3) [pre2 > 0],  g1 = (W2^T g2) [pre1 > 0],  dL/dz = W1^T g1
// Five tensor-core GEMMs per tile of M = 128 pixels (tcgen05, kind::f16, fp32 accumulators in
// TMEM), all operands in shared memory:
//     F1: D1 = Z  W1^T     (K = K1, N = N1)     drain: a1 = relu(D1 + b1) -> ACT, mask1 -> regs
//     F2: D2 = A1 W2^T     (K = N1, N = N2)
//     B1: D3 = G3 W3       (K = Nk, N = N2)     drain: g2 = (D2 + b2 > 0) ? D3 : 0 -> ACT
//     B2: D4 = G2 W2       (K = N2, N = N1)     drain: g1 = mask1 ? D4 : 0 -> ACT
//     B3: D5 = G1 W1       (K = N1, N = K1)     drain: dL/dz -> global
// Two variants. k_mlp_backward (resident, one CTA per SM, used when everything fits):
// the weights are resident in shared memory for the whole persistent launch, each stored ONCE as
// a K-major fp16 tile; B2 and B3 read W2 and W1 transposed through the descriptor's B-major bit
// (an 8x8 core matrix that is K-major for W is MN-major for W^T: LBO and SBO swap roles). One
// activation buffer (ACT, [128][max K] fp16) carries z, a1, g3, g2 and g1 in turn (each GEMM
// completes before its A operand is overwritten). The forward masks are recomputed (two of the
// five GEMMs) rather than stored by the forward pass. k_mlp_backward_s (streamed, two CTAs per
// SM, any MLP the render accepts — e.g. 33-256-256-100): see its comment below.
//
// Biases: when every layer input has two spare padding columns (n_in + 2 <= K1, h1 + 2 <= N1),
// they ride in the GEMMs as fp16 hi/lo pairs on constant-1 inputs, as in the render kernel
// (kFold: z columns n_in, n_in + 1 = 1; W1 rows h1, h1 + 1 make a1 columns h1, h1 + 1 = 1). The
// transposed products then also carry those columns (D4 at h1, h1 + 1 and D5 at n_in, n_in + 1):
// they land in dL/dz channels >= n_in only, which are never stored. Otherwise the drains add
// the fp32 biases.
// 512 threads: 4 per pixel row (TMEM lane), each owning every 4th 16-column group.
// Precision (reading N5): fp16 operands (RN), fp32 accumulation, as the render kernel.
// dL/dbeta is scaled per pixel by an exact power of two before the fp16 rounding (the chain is
// linear in g3 and the masks do not depend on it), so its range never under- or overflows fp16;
// dL/dz is scaled back by the inverse power. The ReLU masks are decided on fp32 accumulators of
// fp16 operands (pre > 0), as the oracle's mask_precision="fp16" mode decides them.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sm100.cuh"

namespace p2s {

struct MlpbParams {
  const float* z;       // [B][n_in][HW] fp32 (the zernike field)
  const float* gb;      // [B][K][HW] fp32 dL/dbeta
  float* gz;            // [B][n_in][HW] fp32 dL/dz (output)
  const uint8_t* wpack; // [W1 | W2 | W3^T | b1 (N1 fp32) | b2 (N2 fp32)], copied to smem offset 0
  int B, HW, n_in, K;
  int K1, N1, N2, Nk;   // padded (multiples of 16) input / hidden / hidden / output widths
  int tiles_per_frame, ntiles;
  int off_w2, off_w3, off_bias, wbytes;  // byte offsets in wpack (= in shared memory)
  int off_act, off_bar;
  int col_b, col_c;     // resident variant: TMEM columns of the RB / RC accumulator regions
  int off_z;            // resident variant: the z tile's own buffer (0: z goes into ACT)
  const float* b3;      // k_mlp_forward: fp32 b3 [K] (read through L1)
  float* beta;          // k_mlp_forward: [B][K][HW] fp32 beta (output)
  // streamed variant (k_mlp_backward_s): the slab table and the ring (B3's W1^T K'-steps are
  // small, K1 x 32 B: g3 of them share one slot, contiguous in W1's layout)
  const uint8_t* ring_src;
  int off_ring, nring, slab_stride, g3;
};

// resident variant: 16 drain warps (4 per TMEM lane quadrant) + the UMMA issuer (warp 16)
constexpr int kMbDrainWarps = 16;
constexpr int kMbThreads = 32 * (kMbDrainWarps + 1);

namespace mlpb {

// D[128 x N] = A[128 x 16 nks] * B^T, A = ACT (K-major, kd = 16 nks), B at b_s:
//   K-major B [N][16 nks]:            lbo = 128,       sbo = 16 * 16 nks, kstep = 256
//   transposed B (stored [16 nks][N]): lbo = 16 * N,    sbo = 128,         kstep = 32 * N, idesc bit 16
P2S_DEV void gemm(uint32_t d, uint32_t a_s, int nks, uint32_t b_s, uint32_t b_lbo, uint32_t b_sbo,
                  uint32_t b_kstep, uint32_t idesc) {
  const uint32_t a_sbo = (uint32_t)nks * 256u;
  for (int ks = 0; ks < nks; ++ks)
    umma_f16_elect(d, sdesc(a_s + (uint32_t)ks * 256u, 128u, a_sbo),
                   sdesc(b_s + (uint32_t)ks * b_kstep, b_lbo, b_sbo), idesc, ks > 0 ? 1u : 0u);
}

// this thread's row of a K-major [128][kd] fp16 tile: element (m, k) at
// (m%8)*16 + (m/8)*kd*16 + (k%8)*2 + (k/8)*128
P2S_DEV uint8_t* row_of(uint8_t* act, int m, int kd) { return act + (m & 7) * 16 + (m >> 3) * kd * 16; }

P2S_DEV void st8(uint8_t* row, int kchunk, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  *reinterpret_cast<uint4*>(row + kchunk * 128) = make_uint4(a, b, c, d);
}
P2S_DEV void st8f(uint8_t* row, int kchunk, const float* v) {
  st8(row, kchunk, pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]), pack_half2(v[6], v[7]));
}
P2S_DEV uint32_t relu2(float a, float b) {  // fp16x2 {lo = relu(a), hi = relu(b)}, RN
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// D[128 x N] = ACT * B^T with each 16-wide K-step of B taken from the next ring slot
// (K-major slabs: lbo 128, sbo 256; W1^T slabs: lbo 16 K1, sbo 128); each slot is released to the
// producer by a commit once the UMMA reading it completes
// (per_slot K-steps per ring slot, kstep bytes apart inside it)
P2S_DEV void gemm_ring(uint32_t d, uint32_t a_s, int nks, uint32_t ring_s, uint32_t stride, uint32_t b_lbo,
                       uint32_t b_sbo, uint32_t idesc, uint64_t* full, uint64_t* empty, int nring, int& s,
                       uint32_t& ph, int per_slot = 1, uint32_t kstep = 0) {
  const uint32_t a_sbo = (uint32_t)nks * 256u;
  for (int k0 = 0; k0 < nks; k0 += per_slot) {
    mbar_wait(&full[s], ph);
    tc_fence_after();
    const int k1 = min(nks, k0 + per_slot);
    for (int ks = k0; ks < k1; ++ks)
      umma_f16_elect(d, sdesc(a_s + (uint32_t)ks * 256u, 128u, a_sbo),
                     sdesc(ring_s + (uint32_t)s * stride + (uint32_t)(ks - k0) * kstep, b_lbo, b_sbo), idesc,
                     ks > 0 ? 1u : 0u);
    umma_commit_elect(&empty[s]);
    if (++s == nring) { s = 0; ph ^= 1; }
  }
}

// barrier among the 16 drain warps only (the issuer warp never joins it)
P2S_DEV void named_sync_drains() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kMbDrainWarps) : "memory"); }

// the CTA's generic-proxy writes to ACT / its TMEM reads are ordered before the next UMMA
P2S_DEV void publish() {
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
}

}  // namespace mlpb

// 8 channels (nvalid real, the rest 0) of one pixel, `stride` floats apart, by a running pointer
// (the drains are issue-bound: per-load offset products and bound checks cost ~2 instructions
// each over the whole tile; full chunks take the unpredicated path)
P2S_DEV void load8(const float* ptr, size_t stride, int nvalid, float (&v)[8]) {
  if (nvalid >= 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j, ptr += stride) v[j] = __ldcs(ptr);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j, ptr += stride) v[j] = j < nvalid ? __ldcs(ptr) : 0.f;
  }
}
// 16 channels (nvalid real, the rest 0) of one pixel, strideB bytes apart (a warp-uniform 64-bit
// increment per load: two integer instructions instead of an index product and a shift)
P2S_DEV void load16b(const float* ptr, size_t strideB, int nvalid, float* v) {
  const char* c = reinterpret_cast<const char*>(ptr);
  if (nvalid >= 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = __ldcs(reinterpret_cast<const float*>(c));
      asm volatile("" : "+l"(c));  // one running pointer (no precomputed address per load)
      c += strideB;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j, c += strideB) v[j] = j < nvalid ? __ldcs(reinterpret_cast<const float*>(c)) : 0.f;
  }
}
// 16 fp32 values -> bits j = [v_j >= +0] (sign bits by two 8-deep funnel-shift chains)
P2S_DEV uint32_t nonneg_bits16(const float (&v)[16]) {
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    lo = __funnelshift_l(__float_as_uint(v[j]), lo, 1);
    hi = __funnelshift_l(__float_as_uint(v[j + 8]), hi, 1);
  }
  return ~(lo | (hi << 8)) & 0xffffu;
}

template <bool kFold>
__global__ void __launch_bounds__(kMbThreads, 1) k_mlp_backward(const __grid_constant__ MlpbParams p) {
  using namespace mlpb;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar_w = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* bar_mma = bar_w + 1;                                   // F2, B1, B2, B3 done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_w + 2);
  uint64_t* bar_f1 = bar_w + 3;                                    // F1 done
  uint64_t* bar_rnd = bar_w + 4;                                   // [4] operand-round ring
  float* s_max = reinterpret_cast<float*>(smem + p.off_bar + 64);  // [4][128]
  const float* s_b1 = reinterpret_cast<const float*>(smem + p.off_bias);
  const float* s_b2 = s_b1 + p.N1;
  uint8_t* act = smem + p.off_act;
  const uint32_t act_s = sbase + (uint32_t)p.off_act;
  // z tile: its own buffer when it fits (the next tile's F1 then runs right behind this tile's
  // B3), else the first K1 columns of ACT
  const bool zsep = p.off_z > 0;
  uint8_t* zbuf = zsep ? smem + p.off_z : act;
  const uint32_t z_s = sbase + (uint32_t)(zsep ? p.off_z : p.off_act);
  const int tid = (int)threadIdx.x, warp = (int)warp_id();

  if (tid == 0) {
    mbar_init(bar_w, 1);
    mbar_init(bar_mma, 1);
    mbar_init(bar_f1, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bar_rnd[i], kMbDrainWarps);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // broadcast from lane 0 so that ptxas keeps the UMMA operands on the uniform datapath (no
  // per-UMMA elect loops; tests/test_abi_cpu.py checks the SASS)
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (tid == 0) {
    mbar_arrive_expect_tx(bar_w, (uint32_t)p.wbytes);
    for (int off = 0; off < p.wbytes; off += 32768)
      bulk_g2s(smem + off, p.wpack + off, (uint32_t)min(32768, p.wbytes - off), bar_w);
  }
  // TMEM: RA = [0, N) F1 / B1, RB = [col_b, +N) F2 / B2, RC = [col_c, +K1) B3 (host-checked)
  const uint32_t tRA = tmem, tRB = tmem + (uint32_t)p.col_b, tRC = tmem + (uint32_t)p.col_c;

  if (warp == kMbDrainWarps) {
    // ================= UMMA issuer: every GEMM streams its K-steps as the drains publish the A
    // operand's 16-column groups, four per round (bar_rnd[round % 4])
    const uint32_t id_f1 = idesc_f16(128, (uint32_t)p.N1), id_f2 = idesc_f16(128, (uint32_t)p.N2);
    const uint32_t id_b2 = idesc_f16(128, (uint32_t)p.N1) | (1u << 16);
    const uint32_t id_b3 = idesc_f16(128, (uint32_t)p.K1) | (1u << 16);
    const uint32_t w1_s = sbase, w2_s = sbase + (uint32_t)p.off_w2, w3_s = sbase + (uint32_t)p.off_w3;
    uint32_t rs = 0;
    auto gemm_rounds = [&](uint32_t d, uint32_t a_s, int nks, uint32_t b_s, uint32_t b_lbo, uint32_t b_sbo,
                           uint32_t b_kstep, uint32_t idesc, uint64_t* done) {
      const uint32_t a_sbo = (uint32_t)nks * 256u;
      for (int k0 = 0; k0 < nks; k0 += 4, ++rs) {
        mbar_wait(&bar_rnd[rs & 3u], (rs >> 2) & 1u);
        tc_fence_after();
        const int k1 = min(nks, k0 + 4);
        for (int ks = k0; ks < k1; ++ks)
          umma_f16_elect(d, sdesc(a_s + (uint32_t)ks * 256u, 128u, a_sbo),
                         sdesc(b_s + (uint32_t)ks * b_kstep, b_lbo, b_sbo), idesc, ks > 0 ? 1u : 0u);
      }
      umma_commit_elect(done);
    };
    if ((int)blockIdx.x < p.ntiles) mbar_wait(bar_w, 0);
    for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x) {
      gemm_rounds(tRA, z_s, p.K1 / 16, w1_s, 128u, (uint32_t)p.K1 * 16u, 256u, id_f1, bar_f1);       // F1 <- z
      gemm_rounds(tRB, act_s, p.N1 / 16, w2_s, 128u, (uint32_t)p.N1 * 16u, 256u, id_f2, bar_mma);    // F2 <- a1
      gemm_rounds(tRA, act_s, p.Nk / 16, w3_s, 128u, (uint32_t)p.Nk * 16u, 256u, id_f2, bar_mma);    // B1 <- g3
      gemm_rounds(tRB, act_s, p.N2 / 16, w2_s, (uint32_t)p.N1 * 16u, 128u, (uint32_t)p.N1 * 32u, id_b2,
                  bar_mma);  // B2 <- g2 (W2 transposed)
      gemm_rounds(tRC, act_s, p.N1 / 16, w1_s, (uint32_t)p.K1 * 16u, 128u, (uint32_t)p.K1 * 32u, id_b3,
                  bar_mma);  // B3 <- g1 (W1 transposed)
    }
  } else {
    // ================= drains: 4 threads per pixel row (TMEM lane); thread q of a row owns the
    // 16-column groups g = 4 r + q (round r)
    const int m = tid & 127, q = tid >> 7;
    const uint32_t tq = (uint32_t)(32 * (warp & 3)) << 16;  // this warp's lane quadrant
    const size_t HW = (size_t)p.HW, HWB = HW * 4;
    uint8_t* const row_k1 = row_of(zbuf, m, p.K1);
    uint8_t* const row_n1 = row_of(act, m, p.N1);
    uint8_t* const row_n2 = row_of(act, m, p.N2);
    uint8_t* const row_nk = row_of(act, m, p.Nk);
    const int G1 = p.N1 / 16, G2 = p.N2 / 16, Gk = p.Nk / 16, Gz = p.K1 / 16;
    uint32_t ph = 0, ph1 = 0, rs = 0;
    // publish this warp's part of one round: generic-proxy writes and TMEM reads are ordered
    // before the UMMAs the issuer starts on the round's barrier
    auto round_done = [&] {
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bar_rnd[rs & 3u]);
      ++rs;
    };
    auto wait_mma = [&] {
      mbar_wait(bar_mma, ph);
      ph ^= 1;
      tc_fence_after();
    };
    // tile t = (frame b, tile lt of the frame), advanced by the grid stride without divisions
    int b = (int)blockIdx.x / p.tiles_per_frame, lt = (int)blockIdx.x - b * p.tiles_per_frame;
    auto advance = [&](int& bb, int& ll) {
      ll += (int)gridDim.x;
      while (ll >= p.tiles_per_frame) { ll -= p.tiles_per_frame; ++bb; }
    };
    // z of a tile -> the z buffer (K1 <= 64: one round; kFold: columns n_in, n_in + 1 = 1)
    float zv[16];
    auto load_z16 = [&](int bb, int ll) {
      const int px = min(ll * 128 + m, p.HW - 1);
      load16b(p.z + (size_t)bb * p.n_in * HW + px + (size_t)(q * 16) * HW, HWB, p.n_in - q * 16, zv);
    };
    auto store_z = [&] {
      if (q < Gz) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int ch = q * 16 + j;
          if (ch >= p.n_in) zv[j] = (kFold && ch < p.n_in + 2) ? 1.f : 0.f;
        }
        st8f(row_k1, 2 * q, zv);
        st8f(row_k1, 2 * q + 1, zv + 8);
      }
      round_done();
    };
    load_z16(b, lt);
    store_z();
    if (!kFold) mbar_wait(bar_w, 0);  // the fp32 biases the drains add
    for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x) {
      const int px = lt * 128 + m;
      const bool valid = px < p.HW;
      const int pxc = valid ? px : p.HW - 1;
      int bn = b, ltn = lt;
      advance(bn, ltn);
      const bool more = t + (int)gridDim.x < p.ntiles;
      if (more) {  // L2 prefetch of the next tile's dL/dbeta rows (4 lines of 128 B per channel)
        const int p0 = ltn * 128;
        const float* gn = p.gb + (size_t)bn * p.K * HW + p0;
        for (int r = tid; r < 4 * p.K; r += kMbDrainWarps * 32) {
          const int qq = p0 + (r & 3) * 32;
          if (qq < p.HW) prefetch_l2(gn + (size_t)(r >> 2) * HW + (r & 3) * 32);
        }
      }
      // ---- dL/dbeta of this tile into registers (in flight during F1 / D1 / F2): groups 4 r + q
      // (the two groups' loads in two batches, the second during D1: 32 loads per thread at once
      // back up the load/store queue)
      float gv[2][16];
      const float* gbb = p.gb + (size_t)b * p.K * HW + pxc;
      load16b(gbb + (size_t)(16 * q) * HW, HWB, p.K - 16 * q, gv[0]);
      mbar_wait(bar_f1, ph1);  // F1
      ph1 ^= 1;
      tc_fence_after();
      // ---- D1 (RA): a1 = relu(pre1) -> ACT (N1 columns), mask1 = [pre1 >= +0] sign bits, per round
      uint32_t mask1[2] = {0u, 0u};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int g = 4 * r + q;
        if (4 * r < G1) {
          if (g < G1) {
            float v[16];
            tmem_ld16(tRA + tq + (uint32_t)(g * 16), v);
            tmem_ld_wait();
            if (!kFold) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] += s_b1[g * 16 + j];
            }
            mask1[r >> 1] |= nonneg_bits16(v) << ((r & 1) * 16);
            st8(row_n1, 2 * g, relu2(v[0], v[1]), relu2(v[2], v[3]), relu2(v[4], v[5]), relu2(v[6], v[7]));
            st8(row_n1, 2 * g + 1, relu2(v[8], v[9]), relu2(v[10], v[11]), relu2(v[12], v[13]), relu2(v[14], v[15]));
          }
          round_done();
        }
        if (r == 0) load16b(gbb + (size_t)(16 * (4 + q)) * HW, HWB, p.K - 16 * (4 + q), gv[1]);
      }
      // per-pixel power-of-two scale of dL/dbeta (the four quarters agree through s_max)
      float mx = 0.f;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < 16; ++j) mx = fmaxf(mx, fabsf(gv[r][j]));
      s_max[q * 128 + m] = mx;
      named_sync_drains();
      mx = fmaxf(fmaxf(s_max[m], s_max[128 + m]), fmaxf(s_max[256 + m], s_max[384 + m]));
      // mx = f 2^ex with f in [0.5, 1) (normal mx; 0 and subnormals take ex = -126, inf/NaN 129):
      // scale by 2^-ex and back by 2^ex, each as two in-range power-of-two factors (exact)
      const int ex = (int)((__float_as_uint(mx) >> 23) & 0xffu) - 126;
      const int e1 = (-ex) / 2, e2 = -ex - e1;
      wait_mma();  // F2: ACT is free, pre2 in RB
      // ---- scaled dL/dbeta -> ACT (Nk columns), per round: B1 streams on them
      {
        const float s1 = exp2i(e1), s2 = exp2i(e2);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int g = 4 * r + q;
          if (4 * r < Gk) {
            if (g < Gk) {
              float v[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = gv[r][j] * s1 * s2;
              st8f(row_nk, 2 * g, v);
              st8f(row_nk, 2 * g + 1, v + 8);
            }
            round_done();
          }
        }
      }
      // ---- RB (pre2) -> mask2 sign bits while B1 runs (RB is free for B2 after this)
      uint32_t mask2[2] = {0u, 0u};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int g = 4 * r + q;
        if (g < G2) {
          float v[16];
          tmem_ld16(tRB + tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          if (!kFold) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += s_b2[g * 16 + j];
          }
          mask2[r >> 1] |= nonneg_bits16(v) << ((r & 1) * 16);
        }
      }
      wait_mma();  // B1: W3^T g3 in RA
      // ---- D3 (RA): g2 = mask2 ? D3 : 0 -> ACT (N2 columns), per round: B2 streams on them
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int g = 4 * r + q;
        if (4 * r < G2) {
          if (g < G2) {
            float v[16];
            tmem_ld16(tRA + tq + (uint32_t)(g * 16), v);
            tmem_ld_wait();
            const uint32_t bits = mask2[r >> 1] >> ((r & 1) * 16);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = ((bits >> j) & 1u) ? v[j] : 0.f;
            st8f(row_n2, 2 * g, v);
            st8f(row_n2, 2 * g + 1, v + 8);
          }
          round_done();
        }
      }
      if (more) load_z16(bn, ltn);  // next tile's z (in flight during B2 / D4)
      wait_mma();  // B2: W2^T g2 in RB
      // ---- D4 (RB): g1 = mask1 ? D4 : 0 -> ACT (N1 columns), per round: B3 streams on them
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int g = 4 * r + q;
        if (4 * r < G1) {
          if (g < G1) {
            float v[16];
            tmem_ld16(tRB + tq + (uint32_t)(g * 16), v);
            tmem_ld_wait();
            const uint32_t bits = mask1[r >> 1] >> ((r & 1) * 16);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = ((bits >> j) & 1u) ? v[j] : 0.f;
            st8f(row_n1, 2 * g, v);
            st8f(row_n1, 2 * g + 1, v + 8);
          }
          round_done();
        }
      }
      // the next tile's z: with its own buffer now (F1 follows B3 on the tensor core; RA's last
      // reader, D3, is done), else once B3 has read g1 out of ACT
      if (more && zsep) store_z();
      wait_mma();  // B3: W1^T g1 in RC; ACT is free
      if (more && !zsep) store_z();
      // ---- D5 (RC) -> dL/dz, unscaled (coalesced: lanes are consecutive pixels)
      if (q < Gz) {
        const float u1 = exp2i(-e1), u2 = exp2i(-e2);
        float v[16];
        tmem_ld16(tRC + tq + (uint32_t)(q * 16), v);
        tmem_ld_wait();
        if (valid) {
          char* ptr = reinterpret_cast<char*>(p.gz + (size_t)b * p.n_in * HW + px + (size_t)(q * 16) * HW);
          const int nv = p.n_in - q * 16;
          if (nv >= 16) {  // (two in-range power-of-two factors, as the scaling)
#pragma unroll
            for (int j = 0; j < 16; ++j, ptr += HWB) __stcs(reinterpret_cast<float*>(ptr), v[j] * u1 * u2);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j, ptr += HWB)
              if (j < nv) __stcs(reinterpret_cast<float*>(ptr), v[j] * u1 * u2);
          }
        }
      }
      tc_fence_before();  // RC reads before the next tile's B3 (ordered by its D4 rounds)
      b = bn;
      lt = ltn;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// ================================================================================================
// k_mlp_forward: step a1 alone -- beta = W3 relu(W2 relu(W1 z + b1) + b2) + b3 per pixel -- with
// the resident variant's weight pack, threads and round streaming (used by p2s_debug_beta and by
// the sequence mode's beta pass): F1 Z W1^T, F2 A1 W2^T, F3 A2 W3^T (W3^T read
// transposed out of the pack's W3^T tile, like B2 reads W2). TMEM regions X / Y alternate per
// tile (F1 -> X, F2 -> Y, F3 -> X), so the next tile's F1 (into this tile's Y) runs while this
// tile's beta drain reads X. b3 is added in fp32 by the beta drain.
template <bool kFold>
__global__ void __launch_bounds__(kMbThreads, 1) k_mlp_forward(const __grid_constant__ MlpbParams p) {
  using namespace mlpb;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar_w = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* bar_mma = bar_w + 1;  // F2, F3 done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_w + 2);
  uint64_t* bar_f1 = bar_w + 3;   // F1 done
  uint64_t* bar_rnd = bar_w + 4;  // [4] operand-round ring
  const float* s_b1 = reinterpret_cast<const float*>(smem + p.off_bias);
  const float* s_b2 = s_b1 + p.N1;
  uint8_t* act = smem + p.off_act;
  const uint32_t act_s = sbase + (uint32_t)p.off_act;
  const bool zsep = p.off_z > 0;
  uint8_t* zbuf = zsep ? smem + p.off_z : act;
  const uint32_t z_s = sbase + (uint32_t)(zsep ? p.off_z : p.off_act);
  const int tid = (int)threadIdx.x, warp = (int)warp_id();

  if (tid == 0) {
    mbar_init(bar_w, 1);
    mbar_init(bar_mma, 1);
    mbar_init(bar_f1, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bar_rnd[i], kMbDrainWarps);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (tid == 0) {
    mbar_arrive_expect_tx(bar_w, (uint32_t)p.wbytes);
    for (int off = 0; off < p.wbytes; off += 32768)
      bulk_g2s(smem + off, p.wpack + off, (uint32_t)min(32768, p.wbytes - off), bar_w);
  }
  const uint32_t tR0 = tmem, tR1 = tmem + (uint32_t)p.col_b;  // X = tR0 on even tiles of the CTA

  if (warp == kMbDrainWarps) {
    // ================= UMMA issuer
    const uint32_t id_f1 = idesc_f16(128, (uint32_t)p.N1), id_f2 = idesc_f16(128, (uint32_t)p.N2);
    const uint32_t id_f3 = idesc_f16(128, (uint32_t)p.Nk) | (1u << 16);
    const uint32_t w1_s = sbase, w2_s = sbase + (uint32_t)p.off_w2, w3_s = sbase + (uint32_t)p.off_w3;
    uint32_t rs = 0;
    auto gemm_rounds = [&](uint32_t d, uint32_t a_s, int nks, uint32_t b_s, uint32_t b_lbo, uint32_t b_sbo,
                           uint32_t b_kstep, uint32_t idesc, uint64_t* done) {
      const uint32_t a_sbo = (uint32_t)nks * 256u;
      for (int k0 = 0; k0 < nks; k0 += 4, ++rs) {
        mbar_wait(&bar_rnd[rs & 3u], (rs >> 2) & 1u);
        tc_fence_after();
        const int k1 = min(nks, k0 + 4);
        for (int ks = k0; ks < k1; ++ks)
          umma_f16_elect(d, sdesc(a_s + (uint32_t)ks * 256u, 128u, a_sbo),
                         sdesc(b_s + (uint32_t)ks * b_kstep, b_lbo, b_sbo), idesc, ks > 0 ? 1u : 0u);
      }
      umma_commit_elect(done);
    };
    if ((int)blockIdx.x < p.ntiles) mbar_wait(bar_w, 0);
    uint32_t par = 0;
    for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x, par ^= 1u) {
      const uint32_t tX = par ? tR1 : tR0, tY = par ? tR0 : tR1;
      gemm_rounds(tX, z_s, p.K1 / 16, w1_s, 128u, (uint32_t)p.K1 * 16u, 256u, id_f1, bar_f1);     // F1 <- z
      gemm_rounds(tY, act_s, p.N1 / 16, w2_s, 128u, (uint32_t)p.N1 * 16u, 256u, id_f2, bar_mma);  // F2 <- a1
      gemm_rounds(tX, act_s, p.N2 / 16, w3_s, (uint32_t)p.Nk * 16u, 128u, (uint32_t)p.Nk * 32u, id_f3,
                  bar_mma);  // F3 <- a2 (W3^T tile read transposed)
    }
  } else {
    // ================= drains (4 threads per pixel row, groups 4 r + q)
    const int m = tid & 127, q = tid >> 7;
    const uint32_t tq = (uint32_t)(32 * (warp & 3)) << 16;
    const size_t HW = (size_t)p.HW, HWB = HW * 4;
    uint8_t* const row_k1 = row_of(zbuf, m, p.K1);
    uint8_t* const row_n1 = row_of(act, m, p.N1);
    uint8_t* const row_n2 = row_of(act, m, p.N2);
    const int G1 = p.N1 / 16, G2 = p.N2 / 16, Gk = p.Nk / 16, Gz = p.K1 / 16;
    uint32_t ph = 0, ph1 = 0, rs = 0, par = 0;
    auto round_done = [&] {
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bar_rnd[rs & 3u]);
      ++rs;
    };
    auto wait_mma = [&] {
      mbar_wait(bar_mma, ph);
      ph ^= 1;
      tc_fence_after();
    };
    int b = (int)blockIdx.x / p.tiles_per_frame, lt = (int)blockIdx.x - b * p.tiles_per_frame;
    auto advance = [&](int& bb, int& ll) {
      ll += (int)gridDim.x;
      while (ll >= p.tiles_per_frame) { ll -= p.tiles_per_frame; ++bb; }
    };
    float zv[16];
    auto load_z16 = [&](int bb, int ll) {
      const int px = min(ll * 128 + m, p.HW - 1);
      load16b(p.z + (size_t)bb * p.n_in * HW + px + (size_t)(q * 16) * HW, HWB, p.n_in - q * 16, zv);
    };
    auto store_z = [&] {
      if (q < Gz) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int ch = q * 16 + j;
          if (ch >= p.n_in) zv[j] = (kFold && ch < p.n_in + 2) ? 1.f : 0.f;
        }
        st8f(row_k1, 2 * q, zv);
        st8f(row_k1, 2 * q + 1, zv + 8);
      }
      round_done();
    };
    // one relu drain of a TMEM region into the ACT columns of the next GEMM, per round
    auto relu_drain = [&](uint32_t tr, int G, uint8_t* row, const float* bias) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int g = 4 * r + q;
        if (4 * r < G) {
          if (g < G) {
            float v[16];
            tmem_ld16(tr + tq + (uint32_t)(g * 16), v);
            tmem_ld_wait();
            if (!kFold) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] += bias[g * 16 + j];
            }
            st8(row, 2 * g, relu2(v[0], v[1]), relu2(v[2], v[3]), relu2(v[4], v[5]), relu2(v[6], v[7]));
            st8(row, 2 * g + 1, relu2(v[8], v[9]), relu2(v[10], v[11]), relu2(v[12], v[13]), relu2(v[14], v[15]));
          }
          round_done();
        }
      }
    };
    load_z16(b, lt);
    store_z();
    if (!kFold) mbar_wait(bar_w, 0);  // the fp32 biases the drains add
    for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x, par ^= 1u) {
      const uint32_t tX = par ? tR1 : tR0, tY = par ? tR0 : tR1;
      const int px = lt * 128 + m;
      const bool valid = px < p.HW;
      int bn = b, ltn = lt;
      advance(bn, ltn);
      const bool more = t + (int)gridDim.x < p.ntiles;
      mbar_wait(bar_f1, ph1);  // F1
      ph1 ^= 1;
      tc_fence_after();
      relu_drain(tX, G1, row_n1, s_b1);  // a1 -> ACT (F2 streams on it)
      if (more) load_z16(bn, ltn);        // next tile's z (in flight during F2 / D2)
      wait_mma();                         // F2: ACT is free
      relu_drain(tY, G2, row_n2, s_b2);  // a2 -> ACT (F3 streams on it)
      if (more && zsep) store_z();        // the next tile's F1 (into Y) runs behind F3
      wait_mma();                         // F3: beta in X; ACT is free
      if (more && !zsep) store_z();
      // ---- beta = D3 + b3 -> global [b][k][px] (K real columns; coalesced: lanes are pixels)
      float* ob = p.beta + (size_t)b * p.K * HW + px;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int g = 4 * r + q;
        if (g < Gk) {
          float v[16];
          tmem_ld16(tX + tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          if (valid) {
            char* ptr = reinterpret_cast<char*>(ob + (size_t)(g * 16) * HW);
            const int nv = p.K - g * 16;
#pragma unroll
            for (int j = 0; j < 16; ++j, ptr += HWB)
              if (j < nv) __stcs(reinterpret_cast<float*>(ptr), v[j] + __ldg(p.b3 + g * 16 + j));
          }
        }
      }
      tc_fence_before();  // X reads before the next tile's F2 (ordered by its D1 rounds)
      b = bn;
      lt = ltn;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// ================================================================================================
// k_mlp_backward_s: the streamed variant — no resident weights, TWO CTAs per SM. Each CTA keeps one
// 256-column TMEM region (the layer-2 mask is taken to bits when D2 is drained, so D3 can reuse the
// region), one activation tile, and a ring fed by a producer warp with every GEMM's weight slabs
// in the fixed per-tile order
//     [F1: W1 K-slabs | F2: W2 K-slabs | B1: W3^T K-slabs | B2: W2 row pairs (W2^T K'-slabs) |
//      B3: W1 row pairs (W1^T K'-slabs), g3 per slot]
// from an L2-resident table. The serial GEMM -> drain chain of one CTA overlaps the other CTA's.
// 288 threads: 8 drain warps (2 threads per TMEM lane, each half of the 16-column groups) + the
// producer (warp 8). Slabs: K-slabs [N][16] (lbo 128, sbo 256); row pairs as stored in the K-major
// [rows][kd] layout (lbo 16 kd, sbo 128, B-major bit).
constexpr int kMbsThreads = 288;

template <bool kFold>
__global__ void __launch_bounds__(kMbsThreads, 2) k_mlp_backward_s(const __grid_constant__ MlpbParams p) {
  using namespace mlpb;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar_mma = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_mma + 1);
  uint64_t* ring_full = bar_mma + 2;  // [<= 16]
  uint64_t* ring_empty = ring_full + 16;
  float* s_max = reinterpret_cast<float*>(smem + p.off_bar + 288);  // [2][128]
  const float* s_b1 = reinterpret_cast<const float*>(smem + p.off_bias);
  const float* s_b2 = s_b1 + p.N1;
  uint8_t* act = smem + p.off_act;
  const uint32_t act_s = sbase + (uint32_t)p.off_act;
  const int tid = (int)threadIdx.x, warp = (int)warp_id();
  const int m = tid & 127, hh = (tid >> 7) & 1;  // pixel row (TMEM lane) and column half

  if (tid == 0) {
    mbar_init(bar_mma, 1);
    for (int i = 0; i < p.nring; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (!kFold)  // fp32 biases for the drains (folded biases ride in the GEMMs)
    for (int i = tid; i < p.N1 + p.N2; i += kMbsThreads)
      const_cast<float*>(s_b1)[i] = reinterpret_cast<const float*>(p.wpack)[i];
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp == 8) {
    // ---- producer: every tile's slab sequence, one bulk copy per slot
    if (lane_id() == 0) {
      const int n1 = p.K1 / 16, n2 = n1 + p.N1 / 16, n3 = n2 + p.Nk / 16, n4 = n3 + p.N2 / 16, nb3 = p.N1 / 16;
      const int nsl = n4 + (nb3 + p.g3 - 1) / p.g3;
      int s = 0;
      uint32_t ph = 0;
      for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x)
        for (int i = 0; i < nsl; ++i) {
          mbar_wait(&ring_empty[s], ph ^ 1);
          const uint32_t bytes =
              (uint32_t)(i < n1 ? p.N1 * 32
                                : (i < n3 ? p.N2 * 32 : (i < n4 ? p.N1 * 32 : min(p.g3, nb3 - p.g3 * (i - n4)) * p.K1 * 32)));
          mbar_arrive_expect_tx(&ring_full[s], bytes);
          bulk_g2s(smem + p.off_ring + s * p.slab_stride, p.ring_src + (size_t)i * p.slab_stride, bytes, &ring_full[s]);
          if (++s == p.nring) { s = 0; ph ^= 1; }
        }
    }
    __syncwarp();
  } else {
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const uint32_t ring_s = sbase + (uint32_t)p.off_ring, stride = (uint32_t)p.slab_stride;
    const uint32_t id_f1 = idesc_f16(128, (uint32_t)p.N1), id_f2 = idesc_f16(128, (uint32_t)p.N2);
    const uint32_t id_b2 = idesc_f16(128, (uint32_t)p.N1) | (1u << 16);
    const uint32_t id_b3 = idesc_f16(128, (uint32_t)p.K1) | (1u << 16);
    const size_t HW = (size_t)p.HW;
    uint8_t* const row_k1 = row_of(act, m, p.K1);
    uint8_t* const row_n1 = row_of(act, m, p.N1);
    uint8_t* const row_n2 = row_of(act, m, p.N2);
    uint8_t* const row_nk = row_of(act, m, p.Nk);
    int rs = 0;
    uint32_t rph = 0, ph = 0;
    auto sync8 = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
    auto publish8 = [&] {
      fence_proxy_async_smem();
      tc_fence_before();
      sync8();
    };
    auto wait_mma = [&] {
      mbar_wait(bar_mma, ph);
      ph ^= 1;
      tc_fence_after();
    };
    for (int t = (int)blockIdx.x; t < p.ntiles; t += (int)gridDim.x) {
      const int b = t / p.tiles_per_frame;
      const int px = (t - b * p.tiles_per_frame) * 128 + m;
      const bool valid = px < p.HW;
      const int pxc = valid ? px : p.HW - 1;
      // ---- z -> ACT (K1 columns; kFold: columns n_in, n_in + 1 = 1)
      {
        const float* zb = p.z + (size_t)b * p.n_in * HW + pxc;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = 2 * i + hh;
          if (c * 8 < p.K1) {
            float v[8];
            load8(zb + (size_t)(c * 8) * HW, HW, p.n_in - c * 8, v);
            if (kFold)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int ch = c * 8 + j;
                if (ch >= p.n_in && ch < p.n_in + 2) v[j] = 1.f;
              }
            st8f(row_k1, c, v);
          }
        }
      }
      publish8();
      if (warp == 0) {
        tc_fence_after();
        gemm_ring(tmem, act_s, p.K1 / 16, ring_s, stride, 128u, 256u, id_f1, ring_full, ring_empty, p.nring, rs, rph);
        umma_commit_elect(bar_mma);
      }
      wait_mma();
      // ---- D1: a1 = relu(pre1) -> ACT (N1), mask1 = [pre1 > 0]
      uint32_t mask1[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int g = 2 * i + hh;
        if (g * 16 < p.N1) {
          float v[16];
          tmem_ld16(tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          if (!kFold) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += s_b1[g * 16 + j];
          }
          uint32_t bits = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) bits |= (v[j] > 0.f ? 1u : 0u) << j;
          mask1[i >> 1] |= bits << ((i & 1) * 16);
          st8(row_n1, 2 * g, relu2(v[0], v[1]), relu2(v[2], v[3]), relu2(v[4], v[5]), relu2(v[6], v[7]));
          st8(row_n1, 2 * g + 1, relu2(v[8], v[9]), relu2(v[10], v[11]), relu2(v[12], v[13]), relu2(v[14], v[15]));
        }
      }
      publish8();
      if (warp == 0) {
        tc_fence_after();
        gemm_ring(tmem, act_s, p.N1 / 16, ring_s, stride, 128u, 256u, id_f2, ring_full, ring_empty, p.nring, rs, rph);
        umma_commit_elect(bar_mma);
      }
      // dL/dbeta of this tile (in flight during F2) and its per-pixel exponent
      float gv[8][8];
      {
        const float* gbb = p.gb + (size_t)b * p.K * HW + pxc;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = 2 * i + hh;
          load8(gbb + (size_t)(c * 8) * HW, HW, p.K - c * 8, gv[i]);
        }
      }
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) mx = fmaxf(mx, fabsf(gv[i][j]));
      s_max[hh * 128 + m] = mx;
      wait_mma();  // F2 done: ACT is free, D2 in the region
      // ---- D2: mask2 = [pre2 > 0] bits (the region is then free for D3)
      uint32_t mask2[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int g = 2 * i + hh;
        if (g * 16 < p.N2) {
          float v[16];
          tmem_ld16(tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          uint32_t bits = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) bits |= (v[j] + (kFold ? 0.f : s_b2[g * 16 + j]) > 0.f ? 1u : 0u) << j;
          mask2[i >> 1] |= bits << ((i & 1) * 16);
        }
      }
      sync8();  // s_max of both halves
      mx = fmaxf(s_max[m], s_max[128 + m]);
      const int ex = (int)((__float_as_uint(mx) >> 23) & 0xffu) - 126;
      const int e1 = (-ex) / 2;
      {
        const float s1 = exp2i(e1), s2 = exp2i(-ex - e1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = 2 * i + hh;
          if (c * 8 < p.Nk) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = gv[i][j] * s1 * s2;
            st8f(row_nk, c, v);
          }
        }
      }
      publish8();
      if (warp == 0) {
        tc_fence_after();
        gemm_ring(tmem, act_s, p.Nk / 16, ring_s, stride, 128u, 256u, id_f2, ring_full, ring_empty, p.nring, rs, rph);
        umma_commit_elect(bar_mma);
      }
      wait_mma();
      // ---- D3 (W3^T g3): g2 = mask2 ? D3 : 0 -> ACT (N2)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int g = 2 * i + hh;
        if (g * 16 < p.N2) {
          float v[16];
          tmem_ld16(tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          const uint32_t bits = mask2[i >> 1] >> ((i & 1) * 16);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = ((bits >> j) & 1u) ? v[j] : 0.f;
          st8f(row_n2, 2 * g, v);
          st8f(row_n2, 2 * g + 1, v + 8);
        }
      }
      publish8();
      if (warp == 0) {
        tc_fence_after();
        gemm_ring(tmem, act_s, p.N2 / 16, ring_s, stride, (uint32_t)p.N1 * 16u, 128u, id_b2, ring_full, ring_empty,
                  p.nring, rs, rph);
        umma_commit_elect(bar_mma);
      }
      wait_mma();
      // ---- D4 (W2^T g2): g1 = mask1 ? D4 : 0 -> ACT (N1)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int g = 2 * i + hh;
        if (g * 16 < p.N1) {
          float v[16];
          tmem_ld16(tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          const uint32_t bits = mask1[i >> 1] >> ((i & 1) * 16);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = ((bits >> j) & 1u) ? v[j] : 0.f;
          st8f(row_n1, 2 * g, v);
          st8f(row_n1, 2 * g + 1, v + 8);
        }
      }
      publish8();
      if (warp == 0) {
        tc_fence_after();
        gemm_ring(tmem, act_s, p.N1 / 16, ring_s, stride, (uint32_t)p.K1 * 16u, 128u, id_b3, ring_full, ring_empty,
                  p.nring, rs, rph, p.g3, (uint32_t)p.K1 * 32u);
        umma_commit_elect(bar_mma);
      }
      wait_mma();
      // ---- D5 (W1^T g1) -> dL/dz, unscaled
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int g = 2 * i + hh;
        if (g * 16 < p.K1) {
          float v[16];
          tmem_ld16(tq + (uint32_t)(g * 16), v);
          tmem_ld_wait();
          if (valid) {
            const float u1 = exp2i(-e1), u2 = exp2i(ex + e1);
            float* ptr = p.gz + (size_t)b * p.n_in * HW + px + (size_t)(g * 16) * HW;
            const int nv = p.n_in - g * 16;
            if (nv >= 16) {
#pragma unroll
              for (int j = 0; j < 16; ++j, ptr += HW) __stcs(ptr, v[j] * u1 * u2);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j, ptr += HW)
                if (j < nv) __stcs(ptr, v[j] * u1 * u2);
            }
          }
        }
      }
      tc_fence_before();  // TMEM reads before the next tile's F1 (ordered by its publish)
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

}  // namespace p2s
