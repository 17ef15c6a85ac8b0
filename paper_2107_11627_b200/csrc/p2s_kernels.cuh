// p2s_kernels.cuh — device side of the P2S hot path (sm_100a).
//
//  k_fused_p2s  steps a0+a1+a2: per pixel tile (128 pixels of one image row per CTA; a CTA
//               pair = one 256-row tcgen05 UMMA tile), the P2S MLP and the
//               K invariant convolutions combined per output pixel (Eq. 5),
//               fp16 operands, fp32 accumulation in TMEM; beta and the K x C convolution
//               results never leave the SM; writes J [B][C][H][W] fp32.
//  k_tilt_warp  step a3: backward bilinear warp with clamp-to-edge.
//
// Layouts:
//  * UMMA operands use the SWIZZLE_NONE K-major canonical layout: element (row, k) at
//    (row%8)*16 + (row/8)*SBO + (k%8)*2 + (k/8)*LBO.
//  * B operands (weight chunks, basis) are pre-packed on the host into 16-K "slabs" split in
//    two row halves (LBO = 128, SBO = 256 -> 16*N bytes per half), in the order the MMA
//    issuer consumes them; each CTA of the pair streams its half (bulk-copy / TMA engine)
//    into a ring of multi-slab stages at the same shared-memory offset.
//  * The convolution A operand (im2col of one input channel) is never materialised per
//    K-step: an 8x-expanded view of the image ("EY" blocks: 8 consecutive rows of one
//    column per 16-byte entry; "EX" rows: 8 consecutive columns of one row) is built once
//    per tile (double-buffered), and each K-step addresses it with an overlapping
//    descriptor (SBO = 16 B per pixel row). See plan_conv() in p2s_host.cu.
//
// Roles (per CTA, 14 warps): w0 TMA producer, w2 UMMA issuer (leader CTA only), w1 w3-5
// builders (A1 = Zernike tile, E views), w6-13 epilogue (2 warpgroups).
// Schedule per tile pair (host-built item list, identical in both CTAs):
//   L1c0 | conv stages | L1c1 | conv stages | L2c0 | ... | L3 | remaining conv stages.
// MLP chunks accumulate in a TMEM "scratch" region next to the C conv accumulators; the
// epilogue warps drain each chunk (bias, ReLU, fp16) into the shared-memory A operand of
// the next layer while the tensor cores run conv stages.
#pragma once
#include <cuda.h>
#include "sm100.cuh"

namespace p2s {

constexpr int kTileM = 128;          // pixels per CTA tile (UMMA M = 256 per CTA pair)
constexpr int kWarpProducer = 0;
// leader CTA: UMMA issuer (idle in the peer). Warp 2 sits on SM sub-partition 2 next to the two
// quadrant-2 epilogue warps only (no builder): issue-slot contention measurably delays UMMA issue.
constexpr int kWarpMma = 2;
constexpr int kNumBuildWarps = 4;
constexpr int kWarpEpi0 = 6;          // warps 6..13
// builder warps are warps 1..5 minus the MMA warp; index 0..3 (-1: not a builder)
__device__ __forceinline__ int builder_index(int warp) {
  return (warp < 1 || warp >= kWarpEpi0 || warp == kWarpMma) ? -1 : (warp < kWarpMma ? warp - 1 : warp - 2);
}
constexpr int kNumEpiWarps = 8;
constexpr int kThreads = 32 * (kWarpEpi0 + kNumEpiWarps);  // 448
constexpr int kBuildThreads = 32 * kNumBuildWarps;
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxConvSteps = 512;
constexpr int kMaxOps = 8;
constexpr int kMaxEy = 16, kMaxEx = 4;
constexpr int kMaxN = 256;           // padded bias vectors

// One ring stage ("item") = nslabs consecutive 16-K slabs of one MLP op or of the conv.
enum ItemFlags : uint8_t { IT_BEGIN = 1, IT_END = 2 };
struct Item {
  uint32_t src_off;      // byte offset of this CTA-rank-0 half in the packed stream
  uint32_t bytes;        // per CTA: nslabs * (16 * N)
  uint32_t half_stride;  // byte offset from the rank-0 half to the rank-1 half
  uint16_t first;        // first K-step (slab) index within the op / conv
  uint16_t nslabs;
  uint8_t kind;          // 0 = MLP op, 1 = conv
  uint8_t op;            // MLP op index
  uint8_t flags;         // IT_BEGIN / IT_END (first / last item of the op or of the conv)
  uint8_t map;           // tensor map (box = one half slab: N/16 rows of 256 B)
  uint8_t rows;          // 256-B rows per half slab (N / 16)
  uint8_t pad[3];
};
static_assert(sizeof(Item) == 24, "Item layout");

// UMMA-issuer view of an item (one LDS.128): A-operand descriptor halves for MLP items (the
// shared-memory base is added on the device), width, dependency waits and commits.
enum MmaItemFlags : uint16_t {
  MI_CONV = 1, MI_WAIT_A1 = 2, MI_WAIT_SCR = 4, MI_WAIT_E = 8,
  MI_COMMIT_A1 = 16, MI_COMMIT_MLP = 32, MI_COMMIT_ACC = 64, MI_WAIT_TMEM = 128,
  MI_COMMIT_E = 256,   // the item is the last reader of its E buffer
  MI_EHALF1 = 512,     // half-E plans: the item reads half 1's buffer (else half 0's)
  MI_WAIT_SCR2 = 1024  // a second SCR_FREE phase (a sequence frame's L1c1: the previous frame's
                       // reduction and this frame's early L1c0 drain)
};
struct MmaItem {
  uint32_t a_lo_rel;   // (smem offset >> 4) | (LBO >> 4) << 16, without the smem base
  uint32_t a_hi;       // SBO >> 4 | version bit
  uint16_t first;      // first K-step (accumulate = first + j > 0; conv step index)
  uint8_t nslabs;
  uint8_t n16;         // N / 16 (UMMA N; B half-slab = N rows/2 * 32 B = 16 N bytes)
  uint16_t flags;
  uint16_t d_col;      // MLP items: TMEM column of the accumulator
};
static_assert(sizeof(MmaItem) == 16, "MmaItem layout");

// One MLP "op" = one output-column chunk of one layer: D[scratch] = A * W[n0:n0+N, :]^T.
struct MlpOp {
  int layer;          // 0, 1, 2
  int n0, N;          // output columns [n0, n0+N) of the layer
  int nks;            // K-steps (input width / 16)
  int first_of_layer, last_of_layer;
  int d_col;          // TMEM column of the accumulator (scratch; a CTA's first tile uses the
                      // still-idle conv accumulator columns for whole-layer L1 / L2 ops)
};

constexpr int kMaxMaps = 6;
struct FusedParams {
  CUtensorMap maps[kMaxMaps];  // the packed B stream as uint8 [rows][256], box {256, N/16}
  const float* image;    // [B][C][H][W]
  const float* zernike;  // [B][n_in][H][W] (NULL when `anchors` is set)
  const float* anchors;  // [B][n_in][G][G] anchor grid: A1 interpolates it
  int G;
  int off_anc, anc_cols;  // shared table of y-interpolated anchor rows [n_in][anc_cols] (per tile)
  float* J;              // [B][C][H][W] (mode 0)
  float* beta_out;       // [B][K][H][W] (mode 1: beta; mode 2: dL/dbeta)
  const float* gJ;  // [B][C][H][W] dL/dJ (the adjoint)
  __half* u_out;    // kAdj = 2: U = beta dL/dJ, fp16 [B][C][K][H][Ws], scaled per (frame, channel)
  const uint32_t* u_maxbits;  // [B][C] float bits of max |dL/dJ| over the plane (k_absmax_planes)
  int Ws;           // U row pitch (ceil8(W))
  int B, C, H, W, n_in;
  int nstrips, ntiles, mode;  // mode 0: MLP + conv -> J ; mode 1: MLP only -> beta ;
                              // mode 2: conv only -> dL/dbeta = sum_c dL/dJ_c C_kc (adjoint)
  int y0, ny;                 // rows [y0, y0 + ny) of every frame (a band of the host path)
  const uint8_t* stream;
  const Item* items;          // [items_full | items_beta | items_first | items_seq]
  int n_items_full, n_items_beta, n_items_first, n_items_seq, n_items_conv;
  int nfr;                    // frames per tile: 1, or a sequence's length (sequence mode: frames
                              // share the image, so each tile's convolutions serve all of them)
  int color;                  // colour mode (per-channel beta): nfr = C passes per tile, pass c
                              // uses Zernike frame b C + c and writes J channel c only
  int tab_cap;                // entries of the shared-memory item tables
  int off_mma, off_steps;     // byte offsets of the MmaItem and conv-step tables
  MlpOp ops[kMaxOps];         // [0, n_ops): per-tile ops; then n_fops whole-layer L1/L2 ops
  int n_ops, n_fops;          // drained in a CTA's first tile instead (mode 0)
  int bias_folded;            // 1: b1..b3 ride in the packed weights (constant-1 padding inputs)
  int l3_hold_ks, hold_k0;    // L3 K-steps [hold_k0, hold_k0 + l3_hold_ks) read the hold buffer
  const MmaItem* mma_items;   // UMMA view of items (same order / modes as `items`)
  const uint32_t* conv_steps; // per conv K-step: descriptor low word (E-relative start>>4 | (LBO>>4)<<16)
  int nconv;
  const float* consts;        // b3[128] svec[128] b1[kMaxN] b2[kMaxN] (zero padded)
  int K, Nk, K1, N1, N2;
  int r, rr;                  // rr = r rounded up to a multiple of 4 (E column origin)
  int n_ey, n_ex, npos_y, npos_x;
  int ey_a0[kMaxEy], ex_a[kMaxEx];
  int chan_bytes;             // E region bytes per channel (buffers are sized for C = 3)
  int n_ebuf;                 // 1 or 2 E buffers
  int ehalf, blkA;            // half-E plan (host plan_conv): buffer h holds tap-row half h of one
                              // tile (EY blocks [0, blkA) | the rest + EX rows), not a whole tile
  int chan_bytes1;            // half-E plans: half 1's per-channel bytes (chan_bytes: half 0's);
                              // buffer 1 starts at 3 chan_bytes (else both are chan_bytes)
  int scr_col;                // TMEM column of beta (L3's output; the MLP scratch start unless mlp_ahead)
  int stage_bytes, nring;
  int off_ring, off_a1, off_a2, off_hold, off_e, off_tab, off_const, off_red, off_bar, smem_bytes;
  int a1_sbo, a2_sbo, hold_sbo;
  unsigned long long* prof;   // P2S_PROFILE builds only: [grid][4][20] cycle counters
  int progressive;            // 1: release beta / each conv accumulator as soon as it is read
  int ecmax;                  // channels the E buffers are sized for (buffer 1 at ecmax chan_bytes)
  int mlp_ahead;              // 1 (one-channel plan): the epilogue drains the next tile's L1 before this
                              // tile's conv epilogue (its L1 / L2 run ahead, beta has its own columns)
};

#ifdef P2S_SLEEP_BUILD
#define WAIT_BUILD(bar, par) mbar_wait_sleep(bar, par, P2S_SLEEP_BUILD)
#else
#define WAIT_BUILD(bar, par) mbar_wait(bar, par)
#endif
#ifdef P2S_SLEEP_EPI
#define WAIT_EPI(bar, par) mbar_wait_sleep(bar, par, P2S_SLEEP_EPI)
#else
#define WAIT_EPI(bar, par) mbar_wait(bar, par)
#endif
#ifdef P2S_SLEEP_PROD
#define WAIT_PROD(bar, par) mbar_wait_sleep(bar, par, P2S_SLEEP_PROD)
#else
#define WAIT_PROD(bar, par) mbar_wait(bar, par)
#endif
// P2S_STARTUP_PROF builds (tools/startup_trace.py): globaltimer stamps of CTA 0's launch phases
#ifdef P2S_STARTUP_PROF
#define STAMP(i) do { if (p.prof && blockIdx.x == 0) p.prof[(i)] = globaltimer_ns(); } while (0)
#define STAMP_CTA(base) do { if (p.prof) p.prof[(base) + blockIdx.x] = globaltimer_ns(); } while (0)
#else
#define STAMP(i) do {} while (0)
#define STAMP_CTA(base) do {} while (0)
#endif
#ifdef P2S_PROFILE
#define PROF_T0() const long long _pt0 = clock64()
#define PROF_ADD(slot) prof_acc[slot] += (unsigned long long)(clock64() - _pt0)
#else
#define PROF_T0() do {} while (0)
#define PROF_ADD(slot) do {} while (0)
#endif

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Barriers marked (L) are used in the leader CTA only and receive arrivals from both CTAs;
// (B) exist in both CTAs and are completed by the leader's multicast UMMA commits; (C) local.
enum Bar {
  BAR_A1_FULL = 0,   // (L) 2 x 4 builder warps
  BAR_A1_EMPTY,      // (B)
  BAR_E_FULL0,       // (L) 2 x 4 builder warps
  BAR_E_FULL1,
  BAR_E_EMPTY0,      // (B)
  BAR_E_EMPTY1,
  BAR_MLP_DONE,      // (B)
  BAR_SCR_FREE,      // (L) 2 x 8 epilogue warps
  BAR_ACC_FULL,      // (B)
  BAR_TMEM_FREE,     // (L) 2 x 8 epilogue warps
  BAR_RING = 10      // then ring_full[n] (L: both CTAs' TMA bytes), ring_empty[n] (B)
};

__device__ __forceinline__ void tile_coords(const FusedParams& p, int t, int& b, int& y, int& x0) {
  const int per_b = p.nstrips * p.ny;
  b = t / per_b;
  const int rem = t - b * per_b;
  const int s = rem / p.ny;
  y = p.y0 + rem - s * p.ny;
  x0 = s * kTileM;
}

// relu(a), relu(b) -> fp16x2 {lo = a, hi = b} in one cvt.rn.relu (RN; equals rn(relu(x)))
__device__ __forceinline__ uint32_t cvt_relu_half2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
// fp32x2 -> fp16x2 (cvt.rn), then max(., 0) in fp16x2
__device__ __forceinline__ uint32_t relu_half2(float2 a) {
  __half2 h = __hmax2(__float22half2_rn(a), __float2half2_rn(0.f));
  return *reinterpret_cast<uint32_t*>(&h);
}

// 8 fp32 image samples -> centred fp16 (x - 0.5 in fp32x2, then cvt.rn to fp16x2)
__device__ __forceinline__ uint32_t centred_half2(float a, float b) {
  __half2 h = __float22half2_rn(__fadd2_rn(make_float2(a, b), make_float2(-0.5f, -0.5f)));
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint4 pack8_centred(const float* v) {
  return make_uint4(centred_half2(v[0], v[1]), centred_half2(v[2], v[3]), centred_half2(v[4], v[5]),
                    centred_half2(v[6], v[7]));
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  return make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
                    pack_half2(v[6], v[7]));
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- im2col view builders
// EY block `blk`: entry i = 8 rows (y - r + a0 + j) at column cx0 + i, centred, fp16.
// EX row `e`:     entry i = 8 columns cx0 + i + j of row (y - r + a), centred, fp16.
// Thread g stores its 4 entries in the order (e + g/2) & 3 so that each quarter-warp
// store covers 128 distinct bytes (bank-conflict free).
// E views of all C channels of one tile. Items of all channels share one loop and each thread
// keeps two items' loads in flight (the build is a chain of L2/HBM round trips).
// EY item (channel c, block blk, group g): 8 rows x 4 columns -> 4 entries of 8 fp16.
__device__ __forceinline__ void load_ey(const FusedParams& p, const float* img, int y, int cx0, int blk, int g,
                                        bool vec, float (&v)[4][8]) {
  const int col0 = cx0 + 4 * g;
  const int ybase = y - p.r + p.ey_a0[blk];
  if (vec && col0 >= 0 && col0 + 3 < p.W) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(img + (size_t)clampi(ybase + j, 0, p.H - 1) * p.W + col0));
      v[0][j] = q.x; v[1][j] = q.y; v[2][j] = q.z; v[3][j] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float* row = img + (size_t)clampi(ybase + j, 0, p.H - 1) * p.W;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e][j] = __ldg(row + clampi(col0 + e, 0, p.W - 1));
    }
  }
}
__device__ __forceinline__ void store_ey(const FusedParams& p, uint8_t* Ec, int blk, int g, const float (&v)[4][8]) {
  uint8_t* dst = Ec + (size_t)blk * p.npos_y * 16 + (size_t)(4 * g) * 16;
  uint4 pk[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) pk[e] = pack8_centred(v[e]);
  const int rot = (g >> 1) & 3;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ee = (e + rot) & 3;  // register select, not a dynamically indexed local array
    const uint4 v01 = (ee & 1) ? pk[1] : pk[0], v23 = (ee & 1) ? pk[3] : pk[2];
    *reinterpret_cast<uint4*>(dst + ee * 16) = (ee & 2) ? v23 : v01;
  }
}
// EX item (channel c, row e, group g): 12 columns of one row -> 4 entries of 8 fp16.
__device__ __forceinline__ void load_ex(const FusedParams& p, const float* img, int y, int cx0, int e, int g,
                                        bool vec, float (&v)[12]) {
  const int col0 = cx0 + 4 * g;
  const float* row = img + (size_t)clampi(y - p.r + p.ex_a[e], 0, p.H - 1) * p.W;
  if (vec && col0 >= 0 && col0 + 11 < p.W) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(row + col0 + 4 * q));
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 12; ++q) v[q] = __ldg(row + clampi(col0 + q, 0, p.W - 1));
  }
}
// Blocks [blk0, blk1) and EX rows [ex0, ex1) of every channel into Eb, block blk0 at offset 0 and
// the EX rows after the blocks (a whole tile: [0, n_ey) / [0, n_ex); a half-E plan: one half).
template <int NT>
__device__ __forceinline__ void build_E_all(const FusedParams& p, uint8_t* Eb, const float* img_b, int y, int x0,
                                            int tid, int blk0, int blk1, int ex0, int ex1, int cstride) {
  const int cx0 = x0 - p.rr;
  const bool vec = (p.W & 3) == 0;
  const size_t HW = (size_t)p.H * p.W;
  const int ngy = p.npos_y >> 2, per_c_y = (blk1 - blk0) * ngy;
  const int tot_y = p.C * per_c_y;
  for (int w = tid; w < tot_y; w += 2 * NT) {
    const int w2 = w + NT;
    const int c0 = w / per_c_y, r0 = w - c0 * per_c_y, bl0 = r0 / ngy, g0 = r0 - bl0 * ngy;
    float v0[4][8], v1[4][8];
    load_ey(p, img_b + c0 * HW, y, cx0, blk0 + bl0, g0, vec, v0);
    int c1 = 0, bl1 = 0, g1 = 0;
    if (w2 < tot_y) {
      c1 = w2 / per_c_y;
      const int r1 = w2 - c1 * per_c_y;
      bl1 = r1 / ngy;
      g1 = r1 - bl1 * ngy;
      load_ey(p, img_b + c1 * HW, y, cx0, blk0 + bl1, g1, vec, v1);
    }
    store_ey(p, Eb + (size_t)c0 * cstride, bl0, g0, v0);
    if (w2 < tot_y) store_ey(p, Eb + (size_t)c1 * cstride, bl1, g1, v1);
  }
  const int ngx = p.npos_x >> 2, per_c_x = (ex1 - ex0) * ngx;
  const int tot_x = p.C * per_c_x;
  const size_t xoff = (size_t)(blk1 - blk0) * p.npos_y * 16;
  for (int w = tid; w < tot_x; w += 2 * NT) {
    const int w2 = w + NT;
    const int c0 = w / per_c_x, r0 = w - c0 * per_c_x, e0 = r0 / ngx, g0 = r0 - e0 * ngx;
    float v0[12], v1[12];
    load_ex(p, img_b + c0 * HW, y, cx0, ex0 + e0, g0, vec, v0);
    int c1 = 0, e1 = 0, g1 = 0;
    if (w2 < tot_x) {
      c1 = w2 / per_c_x;
      const int r1 = w2 - c1 * per_c_x;
      e1 = r1 / ngx;
      g1 = r1 - e1 * ngx;
      load_ex(p, img_b + c1 * HW, y, cx0, ex0 + e1, g1, vec, v1);
    }
    uint8_t* d0 = Eb + (size_t)c0 * cstride + xoff + (size_t)e0 * p.npos_x * 16 + (size_t)(4 * g0) * 16;
#pragma unroll
    for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(d0 + q * 16) = pack8_centred(v0 + q);
    if (w2 < tot_x) {
      uint8_t* d1 = Eb + (size_t)c1 * cstride + xoff + (size_t)e1 * p.npos_x * 16 + (size_t)(4 * g1) * 16;
#pragma unroll
      for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(d1 + q * 16) = pack8_centred(v1 + q);
    }
  }
}

// One 16-column group of the conv epilogue (Eq. 5 reduction): NC real columns of beta (scratch)
// and of each channel's accumulator, fp32x2 FMAs into jc2 (sum_k beta_k C_k) and bs2
// (sum_k beta_k s_k for the centring term).
// Range of U = beta dL/dJ in fp16: each (frame, channel) plane of U is scaled by 2^s,
// s = 7 - floor(log2 max|dL/dJ|), so the plane's largest |dL/dJ| lands in [128, 256): a loss
// reduced over a frame (dL/dout ~ 1e-7) no longer flushes to fp16 zero and dL/dout ~ 1e5 no
// longer overflows (|U| < 65504 while |beta| < 256); k_adjoint_image multiplies its sums by 2^-s.
// maxbits = the float bits of max|dL/dJ| (0: an all-zero plane, scale 1). Exact powers of two.
P2S_DEV float exp2i(int e) { return __int_as_float((e + 127) << 23); }  // 2^e, e in [-126, 127]
__device__ __forceinline__ int u_scale_exp(uint32_t maxbits) {
  if (maxbits == 0u) return 0;
  const int E = (int)((maxbits >> 23) & 0xffu) - 127;  // floor(log2 max) (subnormals: -127)
  const int s = 7 - E;
  return s < -126 ? -126 : (s > 126 ? 126 : s);  // 2^s and 2^-s both normal floats
}

// max |x| of each of n_planes planes of n floats, as float bits (|x| >= 0 orders like uint32);
// out zeroed by the caller. grid (blocks per plane, n_planes).
__global__ void __launch_bounds__(256) k_absmax_planes(const float* __restrict__ x, size_t n,
                                                        uint32_t* __restrict__ out) {
  const float* xp = x + (size_t)blockIdx.y * n;
  uint32_t m = 0u;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(__ldg(xp + i))));
  m = __reduce_max_sync(0xffffffffu, m);
  __shared__ uint32_t red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    m = __reduce_max_sync(0xffffffffu, m);
    if (threadIdx.x == 0 && m) atomicMax(out + blockIdx.y, m);
  }
}

// adjoint epilogue (mode 2) for NC channels: dL/dbeta_k = sum_c dL/dJ_c C_kc over this warp
// group's 16-column groups; C_kc = C'_kc + 0.5 s_k (C' convolves the centred image, s_k = tap sum)
// (s_k is read through L1 from the global table: using the shared copy here made ptxas drop the
// MMA warp's uniformity in this instantiation -- R2UR.BROADCAST before every UMMA, SASS-checked)
template <int NC>
__device__ __forceinline__ void adj_epi(uint32_t tl, int Nk, int K, int wg, int GK, const float* gJ, size_t HW,
                                        const float* __restrict__ sv, float* out, bool st) {
  float gj[NC], gsum = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    gj[c] = st ? __ldg(gJ + c * HW) : 0.f;
    gsum += gj[c];
  }
  for (int gi = wg; gi < GK; gi += 2) {
    float av[NC][16];
#pragma unroll
    for (int c = 0; c < NC; ++c) tmem_ld16(tl + c * Nk + gi * 16, av[c]);
    tmem_ld_wait();
    if (st)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = gi * 16 + i;
        if (k < K) {
          float v = 0.5f * __ldg(sv + k) * gsum;
#pragma unroll
          for (int c = 0; c < NC; ++c) v = fmaf(gj[c], av[c][i], v);
          out[(size_t)k * HW] = v;
        }
      }
  }
}

// adjoint epilogue with U (kAdj = 2): beta_k (MLP output, + b3 unless folded) and the NC
// channels' conv accumulators per 16-column group ->
//   dL/dbeta_k = sum_c dL/dJ_c (C'_kc + 0.5 s_k)      (if dbeta != nullptr)
//   U_kc       = fp16(beta_k dL/dJ_c)                   (plane (c, k) of the pixel's frame; if u)
//   jc[c] += beta_k C'_kc, bs += beta_k s_k            (this warpgroup's part of J, Eq. 5)
// consts: the global [b3 | s] table (read through L1, as adj_epi). real = x < W (pitch columns
// beyond W store zero U so the TMA view reads zeros there).
template <int NC>
__device__ __forceinline__ void adj_u_epi(uint32_t tl, int scr_col, int Nk, int K, int wg, int GK, const float* gJ,
                                          size_t HW, const float* __restrict__ consts, bool b3_folded, float* dbeta,
                                          __half* u, const uint32_t* umax, size_t plane, bool st, bool real,
                                          float (&jc)[3], float& bs) {
  float gj[NC], gu[NC], gsum = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    gj[c] = (st && real) ? __ldg(gJ + c * HW) : 0.f;
    gu[c] = u ? gj[c] * exp2i(u_scale_exp(__ldg(umax + c))) : 0.f;  // U's per-plane range scale
    gsum += gj[c];
  }
  const float4* b34 = reinterpret_cast<const float4*>(consts);
  const float4* sv4 = reinterpret_cast<const float4*>(consts + 128);
  for (int gi = wg; gi < GK; gi += 2) {
    float bv[16], av[NC][16], sv[16];
    tmem_ld16(tl + scr_col + gi * 16, bv);
#pragma unroll
    for (int c = 0; c < NC; ++c) tmem_ld16(tl + c * Nk + gi * 16, av[c]);
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {  // tap sums (and b3) for the 16 columns, zero past K
      const float4 s4 = __ldg(sv4 + gi * 4 + i4);
      sv[4 * i4] = s4.x; sv[4 * i4 + 1] = s4.y; sv[4 * i4 + 2] = s4.z; sv[4 * i4 + 3] = s4.w;
    }
    tmem_ld_wait();
    if (!b3_folded) {
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) {
        const float4 b4 = __ldg(b34 + gi * 4 + i4);
        bv[4 * i4] += b4.x; bv[4 * i4 + 1] += b4.y; bv[4 * i4 + 2] += b4.z; bv[4 * i4 + 3] += b4.w;
      }
    }
    // J parts: the columns past K carry beta = 0 and s = 0 (zero-padded weights and tables)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      bs = fmaf(bv[i], sv[i], bs);
#pragma unroll
      for (int c = 0; c < NC; ++c) jc[c] = fmaf(bv[i], av[c][i], jc[c]);
    }
#ifdef P2S_ABL_NOUSTORE
    if (st && u && gj[0] == 12345.f) {  // timing-only ablation: no U stores
#else
    if (st && u) {
#endif
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = gi * 16 + i;
        if (k < K) {
#pragma unroll
          for (int c = 0; c < NC; ++c) u[((size_t)c * K + k) * plane] = __float2half_rn(bv[i] * gu[c]);
        }
      }
    }
    if (st && real && dbeta) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = gi * 16 + i;
        if (k < K) {
          float v = 0.5f * sv[i] * gsum;
#pragma unroll
          for (int c = 0; c < NC; ++c) v = fmaf(gj[c], av[c][i], v);
          dbeta[(size_t)k * HW] = v;
        }
      }
    }
  }
}

template <int NC>
__device__ __forceinline__ void conv_epi_group(uint32_t tl, int scr_col, int Nk, int gi, int C,
                                               const float* sB3, const float* sSv, float2 (&jc2)[3],
                                               float2& bs2, bool b3_folded) {
  float bv[NC], av[3][NC];
  tmem_ld_n<NC>(tl + scr_col + gi * 16, bv);
#pragma unroll
  for (int c = 0; c < 3; ++c)
    if (c < C) tmem_ld_n<NC>(tl + c * Nk + gi * 16, av[c]);
  tmem_ld_wait();
  const float4* b34 = reinterpret_cast<const float4*>(sB3 + gi * 16);
  const float4* sv4 = reinterpret_cast<const float4*>(sSv + gi * 16);
#pragma unroll
  for (int i4 = 0; i4 < NC / 4; ++i4) {
#ifdef P2S_ABL_NOEPILDS
    const float4 b3 = make_float4(0.01f * i4, 0.02f, 0.03f, 0.04f), sv = make_float4(0.5f, 0.25f, 0.125f, 1.f);
    (void)b34; (void)sv4;
#else
    const float4 b3 = b34[i4], sv = sv4[i4];
#endif
    const int i = 4 * i4;
    float2 be0 = make_float2(bv[i], bv[i + 1]), be1 = make_float2(bv[i + 2], bv[i + 3]);
    if (!b3_folded) {
      be0 = __fadd2_rn(be0, make_float2(b3.x, b3.y));
      be1 = __fadd2_rn(be1, make_float2(b3.z, b3.w));
    }
    bs2 = __ffma2_rn(be0, make_float2(sv.x, sv.y), bs2);
    bs2 = __ffma2_rn(be1, make_float2(sv.z, sv.w), bs2);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (c < C) {
        jc2[c] = __ffma2_rn(be0, make_float2(av[c][i], av[c][i + 1]), jc2[c]);
        jc2[c] = __ffma2_rn(be1, make_float2(av[c][i + 2], av[c][i + 3]), jc2[c]);
      }
  }
}

// A1 from an anchor grid (registration DESIGN.md N1): pixel
// centre (y+.5, x+.5), anchors at (i H/(G-1), j W/(G-1)); bilinear per mode in fp32, then fp16
// like a dense field. Out of line: it keeps the builders' (rarely used) anchor path from
// costing the shared register allocation of the whole kernel.
__device__ __noinline__ void build_A1_anchors(const FusedParams& p, uint8_t* dst, int b, int y, int x0, int x,
                                              int tid, uint8_t* smem) {
  // anchor grid (registration DESIGN.md N1): pixel centre (y+.5, x+.5),
  // anchors at (i H/(G-1), j W/(G-1)); bilinear per mode in fp32, then fp16 like the field
  const int G = p.G;
  int i0 = 0, j0 = 0;
  float fy = 0.f, fx = 0.f;
  if (G > 1) {
    const float u = (y + 0.5f) * (float)(G - 1) / (float)p.H, vv = (x + 0.5f) * (float)(G - 1) / (float)p.W;
    i0 = min((int)floorf(u), G - 2);
    j0 = min((int)floorf(vv), G - 2);
    fy = u - (float)i0;
    fx = vv - (float)j0;
  }
  const int di = G > 1 ? G : 0, dj = G > 1 ? 1 : 0;
  // anchor columns this tile spans (row weights are the same for the whole tile)
  const int jlo = G > 1 ? min((int)floorf((x0 + 0.5f) * (float)(G - 1) / (float)p.W), G - 2) : 0;
  const int xl = min(x0 + kTileM - 1, p.W - 1);
  const int jhi = G > 1 ? min((int)floorf((xl + 0.5f) * (float)(G - 1) / (float)p.W), G - 2) + 1 : 0;
  const int ncol = jhi - jlo + 1;
  if (ncol <= p.anc_cols) {
    // separable: the builders first form R_k[j] = (1-fy) A_k[i0][j] + fy A_k[i0+1][j] for
    // those columns in shared memory, then each pixel needs 2 loads per mode, not 4
    float* R = reinterpret_cast<float*>(smem + p.off_anc);
    named_bar_sync(3, kBuildThreads);  // the previous tile's readers are done with R
    const float* ab = p.anchors + (size_t)b * p.n_in * G * G + (size_t)i0 * G + jlo;
    for (int e = tid; e < p.n_in * ncol; e += kBuildThreads) {
      const int k = e / ncol, c = e - k * ncol;
      const float* a = ab + (size_t)k * G * G + c;
      R[e] = (1.f - fy) * __ldg(a) + fy * __ldg(a + di);
    }
    named_bar_sync(3, kBuildThreads);
    const float* Rp = R + (j0 - jlo);
    for (int k0 = 0; k0 < p.K1; k0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (k0 + i < p.n_in) {
          const float* r0 = Rp + (k0 + i) * ncol;
          v[i] = (1.f - fx) * r0[0] + fx * r0[dj];
        } else {
          v[i] = (p.bias_folded && k0 + i < p.n_in + 2) ? 1.f : 0.f;
        }
      }
      *reinterpret_cast<uint4*>(dst + (k0 >> 3) * 128) = pack8(v);
      *reinterpret_cast<uint4*>(dst + ((k0 >> 3) + 1) * 128) = pack8(v + 8);
    }
  } else {
    const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx, w10 = fy * (1.f - fx), w11 = fy * fx;
    const float* ap = p.anchors + (size_t)b * p.n_in * G * G + (size_t)i0 * G + j0;
    for (int k0 = 0; k0 < p.K1; k0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (k0 + i < p.n_in) {
          const float* a = ap + (size_t)(k0 + i) * G * G;
          v[i] = w00 * __ldg(a) + w01 * __ldg(a + dj) + w10 * __ldg(a + di) + w11 * __ldg(a + di + dj);
        } else {
          v[i] = (p.bias_folded && k0 + i < p.n_in + 2) ? 1.f : 0.f;
        }
      }
      *reinterpret_cast<uint4*>(dst + (k0 >> 3) * 128) = pack8(v);
      *reinterpret_cast<uint4*>(dst + ((k0 >> 3) + 1) * 128) = pack8(v + 8);
    }
  }
}

// kAnchors: Zernike input from an anchor grid (p.anchors) instead of a dense field. A separate
// instantiation: merely having the anchor path in the builders cost the dense kernel ~80 B of
// register spills and ~1.5 % (measured). kAdjoint: mode 2 (conv-only lists, dL/dbeta epilogue),
// likewise its own instantiation; the render instantiations see mode & 1 only (0 or 1).
template <bool kAnchors, int kAdj = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads)
    k_fused_p2s(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* ring_full = bars + BAR_RING;
  uint64_t* ring_empty = bars + BAR_RING + p.nring;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + BAR_RING + 2 * p.nring);
  uint8_t* ring = smem + p.off_ring;
  uint8_t* sA1 = smem + p.off_a1;
  uint8_t* sA2 = smem + p.off_a2;
  uint8_t* sHold = smem + p.off_hold;
  uint8_t* sE = smem + p.off_e;
  Item* sItems = reinterpret_cast<Item*>(smem + p.off_tab);
  MmaItem* sMma = reinterpret_cast<MmaItem*>(smem + p.off_mma);
  uint32_t* sSteps = reinterpret_cast<uint32_t*>(smem + p.off_steps);
  float* sConst = reinterpret_cast<float*>(smem + p.off_const);
  // [b3 | tap sums | b1 | b2]; with folded biases only the first 256 floats are staged
  float* sB3 = sConst;
  float* sSv = sConst + 128;
  float* sB1 = sConst + 256;
  float* sB2 = sConst + 256 + kMaxN;
  float4* sRed = reinterpret_cast<float4*>(smem + p.off_red);  // [2][128] partial J (WG1 -> WG0)

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // per-cluster contiguous range of tile pairs; this CTA takes tile 2*pair + rank
  const int npairs = (p.ntiles + 1) >> 1;
  const int ncl = gridDim.x >> 1, cl = blockIdx.x >> 1;
  const int pr_begin = (int)(((long long)cl * npairs) / ncl);
  const int pr_end = (int)(((long long)(cl + 1) * npairs) / ncl);
  // kAdj 1: dL/dbeta only (conv-only lists, mode 2); kAdj 2: dL/dbeta + U = beta dL/dJ (the
  // render flow, mode 0, with the adjoint epilogue)
  const int pmode = kAdj == 1 ? 2 : (kAdj == 2 ? 0 : (p.mode & 1));
  // per-tile item lists: tile 0 of this CTA uses list A (MLP first), later tiles list B
  const int offC = p.n_items_full + p.n_items_beta + p.n_items_first + p.n_items_seq;  // conv-only list
  const int nA = pmode == 0 ? p.n_items_first : (pmode == 1 ? p.n_items_beta : p.n_items_conv);
  const int nB = pmode == 0 ? p.n_items_full : (pmode == 1 ? p.n_items_beta : p.n_items_conv);
  const int offA = pmode == 0 ? p.n_items_full + p.n_items_beta : (pmode == 1 ? p.n_items_full : offC);
  const int offB = pmode == 0 ? 0 : (pmode == 1 ? p.n_items_full : offC);
  // sequence mode: after a tile's first frame (list A / B), nfr - 1 MLP-only lists S
  const int nS = p.nfr > 1 ? p.n_items_seq : 0;
  const int offS = p.n_items_full + p.n_items_beta + p.n_items_first;
  const int nfr = p.nfr;
  // items of segment (tile it, frame fr) start at table index seg_base, n of them
  auto seg_base = [&](int it, int fr) { return fr > 0 ? nA + nB : (it == 0 ? 0 : nA); };
  auto seg_len = [&](int it, int fr) { return fr > 0 ? nS : (it == 0 ? nA : nB); };
#ifdef P2S_PROFILE
  unsigned long long prof_acc[20];
#pragma unroll
  for (int i = 0; i < 20; ++i) prof_acc[i] = 0;
  const long long prof_start = clock64();
  prof_acc[10] = globaltimer_ns();
#endif

  if (threadIdx.x == 0) { STAMP(0); STAMP_CTA(16); }
  // ---- setup: the item, step and constant tables -> shared memory as 4-byte async copies, all
  // in flight at once (dependent load/store loops cost one global round trip per table)
  {
    constexpr int wi = (int)(sizeof(Item) / 4), wm = (int)(sizeof(MmaItem) / 4);
    const uint32_t* gi = reinterpret_cast<const uint32_t*>(p.items);
    const uint32_t* gm = reinterpret_cast<const uint32_t*>(p.mma_items);
    uint32_t* si = reinterpret_cast<uint32_t*>(sItems);
    uint32_t* sm = reinterpret_cast<uint32_t*>(sMma);
    auto src_of = [&](int i) { return i < nA ? offA + i : (i < nA + nB ? offB + (i - nA) : offS + (i - nA - nB)); };
    for (int w = threadIdx.x; w < (nA + nB + nS) * wi; w += kThreads) {
      const int i = w / wi;
      cp_async4(si + w, gi + (size_t)src_of(i) * wi + (w - i * wi));
    }
    for (int w = threadIdx.x; w < (nA + nB + nS) * wm; w += kThreads) {
      const int i = w / wm;
      cp_async4(sm + w, gm + (size_t)src_of(i) * wm + (w - i * wm));
    }
    for (int i = threadIdx.x; i < p.nconv; i += kThreads) cp_async4(sSteps + i, p.conv_steps + i);
    const int n_const = p.bias_folded ? 256 : 256 + 2 * kMaxN;
    for (int i = threadIdx.x; i < n_const; i += kThreads) cp_async4(sConst + i, p.consts + i);
    cp_async_wait_all();
  }
  if (threadIdx.x == 0) STAMP(1);
  if (threadIdx.x == 0) {
    mbar_init(&bars[BAR_A1_FULL], 2 * kNumBuildWarps);
    mbar_init(&bars[BAR_A1_EMPTY], 1);
    mbar_init(&bars[BAR_E_FULL0], 2 * kNumBuildWarps);
    mbar_init(&bars[BAR_E_FULL1], 2 * kNumBuildWarps);
    mbar_init(&bars[BAR_E_EMPTY0], 1);
    mbar_init(&bars[BAR_E_EMPTY1], 1);
    mbar_init(&bars[BAR_MLP_DONE], 1);
    mbar_init(&bars[BAR_SCR_FREE], 2 * kNumEpiWarps);
    mbar_init(&bars[BAR_ACC_FULL], 1);
    mbar_init(&bars[BAR_TMEM_FREE], 2 * kNumEpiWarps);
    for (int i = 0; i < p.nring; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMma) tmem_alloc2<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers are initialised before any remote arrive
  if (threadIdx.x == 0) STAMP(2);
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpProducer) {
#ifndef P2S_ABL_NOTMA
    // ================= producer: TMA this CTA's half of every slab into the ring; both CTAs'
    // copies complete on the leader's ring_full (the leader arms it with both halves' bytes)
    if (lane == 0) {
      for (int i = 0; i < kMaxMaps; ++i) prefetch_tmap(&p.maps[i]);
      int s = 0;
      uint32_t ph = 0;
      for (int pr = pr_begin; pr < pr_end; ++pr)
      for (int fr = 0; fr < nfr; ++fr) {
        const int n_items = seg_len(pr - pr_begin, fr), base = seg_base(pr - pr_begin, fr);
        for (int g = 0; g < n_items; ++g) {
          const Item it = sItems[base + g];
          { PROF_T0(); WAIT_PROD(&ring_empty[s], ph ^ 1); PROF_ADD(7); }
          if (leader) mbar_arrive_expect_tx(&ring_full[s], 2u * it.bytes);
          const uint32_t mb = cluster_addr(&ring_full[s], 0);
          const int y0 = (int)((it.src_off + rank * it.half_stride) >> 8);
          uint8_t* dst = ring + (size_t)s * p.stage_bytes;
          for (int j = 0; j < it.nslabs; ++j)
            tma2_load_2d(dst + (size_t)j * it.rows * 256, &p.maps[it.map], 0, y0 + j * it.rows, mb);
          if (++s == p.nring) { s = 0; ph ^= 1; }
        }
      }
    }
#endif
  } else if (warp == kWarpMma && leader) {
    // ================= leader: UMMA issuer (whole warp, uniform values; one lane issues) ====
    // Descriptors are assembled from precomputed 32-bit halves so the per-UMMA work is one
    // or two uniform adds: lo = start>>4 | (LBO>>4)<<16, hi = SBO>>4 | version(bit 46).
    const uint32_t ring_lo = (smem_u32(ring) >> 4) | ((128u >> 4) << 16);
    const uint32_t e_lo = smem_u32(sE) >> 4;
    const uint32_t hi_b = (256u >> 4) | (1u << 14);
    const uint32_t hi_conv = (128u >> 4) | (1u << 14);
    const uint32_t id_conv = idesc_f16(256, p.Nk);
    const uint32_t stage16 = (uint32_t)p.stage_bytes >> 4;
    const uint32_t ch16_0 = (uint32_t)p.chan_bytes >> 4, ch16_1 = (uint32_t)p.chan_bytes1 >> 4;
    const uint32_t ebuf16 = (uint32_t)p.ecmax * ch16_0;  // buffer 1's offset
    const int C = p.C, nring = p.nring, ebufs = p.n_ebuf, mode = pmode, ehalf = p.ehalf;
    const uint32_t acc1 = tmem + (uint32_t)p.Nk, acc2 = tmem + 2u * (uint32_t)p.Nk;
    const uint32_t smem_lo = smem_u32(smem) >> 4;
    const uint32_t id_base = idesc_f16(256, 0);
    int s = 0;
    uint32_t ph = 0;
    uint32_t scr_waits = 0, a1_waits = 0;
    uint32_t e_par = 0;  // bit b: phase parity of E buffer b's next use (branch-free: keeps the loop uniform)
    int pending = -1;  // ring slot whose release commit is deferred behind the next UMMAs
#ifdef P2S_PROFILE
    prof_acc[11] = globaltimer_ns();
#endif
    const int ntl = pr_end - pr_begin;
    const int total = ntl > 0 ? nA + (ntl - 1) * nB + ntl * (nfr - 1) * nS : 0;
#ifdef P2S_STARTUP_PROF
    bool stamped_conv = false;
#endif
    MmaItem cur = sMma[0];
    for (int step = 0, it = 0, fr = 0, g = 0; step < total; ++step) {
      const int n_items = seg_len(it, fr);
      // prefetch the next item: same segment, else the next frame's (S) or the next tile's (B)
      const MmaItem nxt = sMma[g + 1 < n_items ? seg_base(it, fr) + g + 1 : (fr + 1 < nfr ? nA + nB : nA)];
      const uint32_t f = cur.flags;
      // E buffer of this item: half-E plans by the item's half, else by tile parity (broadcast
      // from lane 0: a value ptxas cannot prove warp-uniform costs the issue loop its uniform
      // datapath, SASS-checked)
      const int eb = ehalf ? __shfl_sync(0xffffffffu, (f & MI_EHALF1) ? 1 : 0, 0) : (ebufs == 2 ? (it & 1) : 0);
#ifdef P2S_PROFILE
      const long long tr_a = clock64();
#endif
      if (kAdj != 1 && (f & MI_WAIT_A1)) {
        { PROF_T0(); mbar_wait(&bars[BAR_A1_FULL], a1_waits & 1); PROF_ADD(0); }
        ++a1_waits;
      }
      if (f & MI_WAIT_TMEM) { PROF_T0(); mbar_wait(&bars[BAR_TMEM_FREE], (it & 1) ^ 1); PROF_ADD(1); }
      if (kAdj != 1 && (f & MI_WAIT_SCR)) {
        { PROF_T0(); mbar_wait(&bars[BAR_SCR_FREE], scr_waits & 1); PROF_ADD(2); }
        ++scr_waits;
      }
      if (kAdj != 1 && (f & MI_WAIT_SCR2)) {
        mbar_wait(&bars[BAR_SCR_FREE], scr_waits & 1);
        ++scr_waits;
      }
      if (f & MI_WAIT_E) { PROF_T0(); mbar_wait(&bars[BAR_E_FULL0 + eb], (e_par >> eb) & 1u); PROF_ADD(3); }
#ifndef P2S_ABL_NOTMA
      { PROF_T0(); mbar_wait(&ring_full[s], ph); PROF_ADD(5); }
#endif
      tc_fence_after();
#ifdef P2S_STARTUP_PROF
      if (lane == 0 && step == 0) STAMP(5);
      if (lane == 0 && (f & MI_CONV) && !stamped_conv) { STAMP(6); stamped_conv = true; }
#endif
#ifdef P2S_PROFILE
      const long long tr_b = clock64();
#endif
      const uint32_t b_lo0 = ring_lo + (uint32_t)s * stage16;
      const uint32_t n = cur.nslabs;
      const uint32_t half16 = (uint32_t)cur.n16 * 16u;  // (16 * N) >> 4
      const uint32_t first = cur.first;
#if defined(P2S_ABL_NOCONVMMA)
      if ((f & MI_CONV) && n == 0) {
#else
      if (kAdj == 1 || (f & MI_CONV)) {  // (the kAdj = 1 lists hold conv stages only)
#endif
        PROF_T0();
        const uint32_t e0 = e_lo + (uint32_t)eb * ebuf16;
        const uint32_t ch16 = eb ? ch16_1 : ch16_0;  // channel stride of this buffer
        const uint32_t* steps = sSteps + first;
#pragma unroll 2
        for (uint32_t j = 0; j < n; ++j) {
          const uint32_t a_lo = e0 + steps[j];
          const uint64_t bd = ((uint64_t)hi_b << 32) | (b_lo0 + j * half16);
          const uint32_t accum = (first + j) > 0;
          umma2_f16_elect(tmem, ((uint64_t)hi_conv << 32) | a_lo, bd, id_conv, accum);
          if (C > 1) umma2_f16_elect(acc1, ((uint64_t)hi_conv << 32) | (a_lo + ch16), bd, id_conv, accum);
          if (C > 2) umma2_f16_elect(acc2, ((uint64_t)hi_conv << 32) | (a_lo + 2u * ch16), bd, id_conv, accum);
          if (j == 0 && pending >= 0) { umma2_commit_elect(&ring_empty[pending]); pending = -1; }
        }
        PROF_ADD(4);
#if defined(P2S_ABL_NOCONVMMA)
      } else if (!(f & MI_CONV)) {
#else
      } else {
#endif
#ifdef P2S_ABL_NOMLPMMA
        if (n == 0)
#endif
        {
        PROF_T0();
        const uint32_t idesc = id_base | ((uint32_t)cur.n16 << 18);  // N>>3 at bit 17
        const uint32_t a_lo0 = smem_lo + cur.a_lo_rel;
        const uint32_t dacc = tmem + cur.d_col;
#pragma unroll 2
        for (uint32_t j = 0; j < n; ++j) {
          const uint64_t ad = ((uint64_t)cur.a_hi << 32) | (a_lo0 + j * 16u);
          const uint64_t bd = ((uint64_t)hi_b << 32) | (b_lo0 + j * half16);
          umma2_f16_elect(dacc, ad, bd, idesc, (first + j) > 0);
          if (j == 0 && pending >= 0) { umma2_commit_elect(&ring_empty[pending]); pending = -1; }
        }
        PROF_ADD(6);
        }
      }
#if defined(P2S_ABL_NOCONVMMA) || defined(P2S_ABL_NOMLPMMA)
      if (pending >= 0) { umma2_commit_elect(&ring_empty[pending]); pending = -1; }
#endif
      // completion signals for the epilogue / builders are not deferred
      if (f & (MI_COMMIT_A1 | MI_COMMIT_MLP | MI_COMMIT_ACC | MI_COMMIT_E)) {
        umma2_commit_elect(&ring_empty[s]);  // keep ring releases in order before a hand-off
        if (f & MI_COMMIT_A1) umma2_commit_elect(&bars[BAR_A1_EMPTY]);
        if (f & MI_COMMIT_MLP) umma2_commit_elect(&bars[BAR_MLP_DONE]);
        if ((f & MI_COMMIT_E) && mode != 1) {  // the last reader of E buffer eb
          umma2_commit_elect(&bars[BAR_E_EMPTY0 + eb]);
          e_par ^= 1u << eb;
        }
        if (f & MI_COMMIT_ACC) umma2_commit_elect(&bars[BAR_ACC_FULL]);
      } else {
        pending = s;
      }
#ifdef P2S_PROFILE
      if (p.prof && blockIdx.x == 0 && step < 256 && lane == 0) {  // per-item issue timeline
        unsigned long long* tr = p.prof + 148 * 4 * 20 + 4 * step;
        tr[0] = (unsigned long long)(tr_a - prof_start);
        tr[1] = (unsigned long long)(tr_b - prof_start);
        tr[2] = (unsigned long long)(clock64() - prof_start);
        tr[3] = f | ((unsigned long long)cur.nslabs << 16) | ((unsigned long long)cur.n16 << 24);
      }
#endif
      if (++s == nring) { s = 0; ph ^= 1; }
      cur = nxt;
      if (++g == n_items) {
        g = 0;
        if (++fr == nfr) { fr = 0; ++it; }
      }
    }
    if (pending >= 0) umma2_commit_elect(&ring_empty[pending]);
    if (lane == 0) STAMP(10);
  } else if (builder_index(warp) >= 0) {
    // ================= builders: A1 (Zernike tile, fp16) and E views (fp16, centred) =====
    const int tid = builder_index(warp) * 32 + lane;
    const size_t HW = (size_t)p.H * p.W;
    uint32_t e_use0 = 0, e_use1 = 0, a1_builds = 0;
    int it = 0;
    for (int pr = pr_begin; pr < pr_end; ++pr, ++it)
    for (int fr = 0; fr < nfr; ++fr) {
      const int t = min(2 * pr + (int)rank, p.ntiles - 1);  // odd tail: duplicate, not stored
      int b, y, x0;
      tile_coords(p, t, b, y, x0);
      if (pmode != 2) {  // (mode 2, the adjoint, needs only the E views)
        // --- A1 of Zernike frame b nfr + fr (sequence mode: b = 0; colour mode: channel fr): row m =
        //     pixel x0+m, k = Zernike index (zero-padded to K1)
        { PROF_T0(); WAIT_BUILD(&bars[BAR_A1_EMPTY], (a1_builds & 1) ^ 1); PROF_ADD(9); }
        ++a1_builds;
        {
          const int m = tid;
          const int x = min(x0 + m, p.W - 1);
          uint8_t* dst = sA1 + (m & 7) * 16 + (m >> 3) * p.a1_sbo;
          if constexpr (!kAnchors) {
            const float* zp = p.zernike + (size_t)(b * nfr + fr) * p.n_in * HW + (size_t)y * p.W + x;
            for (int k0 = 0; k0 < p.K1; k0 += 16) {
              float v[16];
  #pragma unroll
              for (int i = 0; i < 16; ++i)
                v[i] = (k0 + i < p.n_in) ? __ldg(zp + (size_t)(k0 + i) * HW)
                                         : ((p.bias_folded && k0 + i < p.n_in + 2) ? 1.f : 0.f);
              *reinterpret_cast<uint4*>(dst + (k0 >> 3) * 128) = pack8(v);
              *reinterpret_cast<uint4*>(dst + ((k0 >> 3) + 1) * 128) = pack8(v + 8);
            }
          } else {
            build_A1_anchors(p, dst, b * nfr + fr, y, x0, x, tid, smem);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_A1_FULL], 0);
        if (lane == 0 && builder_index(warp) == 0 && a1_builds == 1) STAMP(3);
      }
      if (pmode == 1 || fr > 0) continue;  // E views: once per tile (every frame shares the image)
      // --- E views of every channel (the CTA's first tile: built by the idle epilogue warps).
      // Half-E plans: buffer h <- half h of this tile, one after the other
      if (it == 0) { ++e_use0; if (p.ehalf) ++e_use1; continue; }
      for (int hh = 0; hh < 1 + p.ehalf; ++hh) {
        const int eb = p.ehalf ? hh : (p.n_ebuf == 2 ? (it & 1) : 0);
        { PROF_T0(); WAIT_BUILD(&bars[BAR_E_EMPTY0 + eb], ((eb ? e_use1 : e_use0) & 1) ^ 1); PROF_ADD(11); }
        if (eb) ++e_use1; else ++e_use0;
        uint8_t* Eb = sE + (size_t)eb * p.ecmax * p.chan_bytes;  // buffers are sized for ecmax channels (half 0 first)
        {
          PROF_T0();
#ifndef P2S_ABL_NOE
          // (one call site: every inlined copy of the builder costs registers the whole kernel shares)
          const bool h0 = p.ehalf && hh == 0, h1 = p.ehalf && hh == 1;
          build_E_all<kBuildThreads>(p, Eb, p.image + (size_t)b * p.C * HW, y, x0, tid, h1 ? p.blkA : 0,
                                     h0 ? p.blkA : p.n_ey, 0, h0 ? 0 : p.n_ex, h1 ? p.chan_bytes1 : p.chan_bytes);
#endif
          PROF_ADD(12);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_E_FULL0 + eb], 0);
      }
    }
  } else if (warp >= kWarpEpi0) {
    // ================= epilogue: two warpgroups split every TMEM drain by 16-col groups =====
    // ---- the CTA's first tile: its E views (E buffer 0) come from the 8 epilogue warps, idle
    // until the first MLP chunk, so the first conv stage does not wait for the builders' A1 + E
    // chain of cold loads. (tile_coords() here, not in the shared prologue: there it cost the
    // UMMA issuer its convergence proof - ptxas then wraps every elect in a loop; test_abi_cpu
    // checks the SASS.)
    if (pr_begin < pr_end && pmode != 1) {
      int b0, y0, xs;
      tile_coords(p, min(2 * pr_begin + (int)rank, p.ntiles - 1), b0, y0, xs);
      const size_t HW0 = (size_t)p.H * p.W;
#ifndef P2S_ABL_NOE
      const int etid = (warp - kWarpEpi0) * 32 + lane;
      for (int hh = 0; hh < 1 + p.ehalf; ++hh) {  // half-E plans: both halves, into buffers 0 and 1
        const bool h0 = p.ehalf && hh == 0, h1 = p.ehalf && hh == 1;
        build_E_all<32 * kNumEpiWarps>(p, sE + (size_t)hh * p.ecmax * p.chan_bytes, p.image + (size_t)b0 * p.C * HW0, y0,
                                       xs, etid, h1 ? p.blkA : 0, h0 ? p.blkA : p.n_ey, 0, h0 ? 0 : p.n_ex,
                                       h1 ? p.chan_bytes1 : p.chan_bytes);
      }
#endif
      fence_proxy_async_smem();
      named_bar_sync(2, 32 * kNumEpiWarps);
      if (warp - kWarpEpi0 < kNumBuildWarps && lane == 0) {
        mbar_arrive_remote(&bars[BAR_E_FULL0], 0);
        if (p.ehalf) mbar_arrive_remote(&bars[BAR_E_FULL1], 0);
      }
      if (warp == kWarpEpi0 && lane == 0) STAMP(4);
    }
    const int ew = warp - kWarpEpi0;        // 0..7
    const int wg = ew >> 2;                 // warpgroup 0 / 1
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;            // pixel (row of every accumulator)
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const size_t HW = (size_t)p.H * p.W;
    const int C = p.C;
    uint32_t mlp_waits = 0;
    uint8_t* a2row = sA2 + (m & 7) * 16 + (m >> 3) * p.a2_sbo;
    uint8_t* hrow = sHold + (m & 7) * 16 + (m >> 3) * p.hold_sbo;
    int it = 0;
    uint32_t acc_waits = 0, red_i = 0;
    for (int pr = pr_begin; pr < pr_end; ++pr, ++it)
    for (int fr = 0; fr < nfr; ++fr) {  // sequence mode: every frame of the tile's image
      const int t_raw = 2 * pr + (int)rank;
      const bool store = t_raw < p.ntiles;
      int b, y, x0;
      tile_coords(p, min(t_raw, p.ntiles - 1), b, y, x0);
      // a CTA's first tile (mode 0) runs L1 and L2 as whole-layer ops (p.ops[n_ops, +n_fops))
      const bool fops = pmode == 0 && it == 0 && fr == 0 && p.n_fops > 0;
      const int o_begin = fops ? p.n_ops : 0, o_end = pmode == 2 ? 0 : (fops ? p.n_ops + p.n_fops : p.n_ops);
      // MLP ahead (one-channel plan, one frame per tile): this tile's L1 was drained in the previous
      // iteration and the next tile's L1 is drained (after this tile's L2) before this tile's conv
      // epilogue, so the tensor core runs the next L2 while the epilogue reads beta and the
      // accumulator. One loop body for every drain (a second inlined copy costs registers).
      // (Sequence frames of an early-L1 plan keep this order: their L1c0 runs during the previous
      // frame's reduction but is drained after it -- draining it first put the A1 build on the
      // epilogue's path, measured slower.)
      const bool ahead = pmode == 0 && nfr == 1 && p.mlp_ahead != 0;
      const int o_stop = o_end + ((ahead && pr + 1 < pr_end) ? 1 : 0);
      for (int k = o_begin; k < o_stop; ++k) {
        const int o = k < o_end ? k : 0;
        if (k < o_end && (p.ops[o].layer == 2 || (ahead && o == 0 && it > 0))) continue;  // (beta stays)
        const MlpOp op = p.ops[o];
        { PROF_T0(); WAIT_EPI(&bars[BAR_MLP_DONE], mlp_waits & 1); PROF_ADD(13); }
        ++mlp_waits;
        tc_fence_after();
#ifdef P2S_PROFILE
        const long long td0 = clock64();
#endif
        const float* bias = (op.layer == 0 ? sB1 : sB2) + op.n0;
        const int G = op.N >> 4;
        // L2 chunks other than the last go to the hold buffer (L3 reads them from there)
        const bool to_hold = op.layer == 1 && !op.last_of_layer;
        uint8_t* dst = to_hold ? hrow : a2row;
        const int kc0 = (to_hold ? 0 : op.n0) >> 3;
#pragma unroll 1
#ifdef P2S_ABL_NODRAIN
        for (int hp = 0; hp < 0; ++hp) {
#else
        for (int hp = 0; hp < 4; ++hp) {     // groups gi = wg + 2*hg, two TMEM loads per wait
#endif
          const int gi0 = wg + 4 * hp, gi1 = gi0 + 2;
          if (gi0 >= G) break;
          float v[2][16];
          tmem_ld16(tl + op.d_col + gi0 * 16, v[0]);
          if (gi1 < G) tmem_ld16(tl + op.d_col + gi1 * 16, v[1]);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int gi = gi0 + 2 * u;
            if (gi < G) {
              uint32_t hv[8];
              if (p.bias_folded) {
                // bias already in the accumulator: one cvt.rn.relu.f16x2 per two values
#pragma unroll
                for (int i2 = 0; i2 < 8; ++i2) hv[i2] = cvt_relu_half2(v[u][2 * i2], v[u][2 * i2 + 1]);
              } else {
                // bias add in packed fp32x2, round to fp16x2 (RN), then ReLU in fp16x2: rounding
                // is monotone and sign-preserving, so relu(rn(x)) == rn(relu(x))
                const float4* b4 = reinterpret_cast<const float4*>(bias + gi * 16);
#pragma unroll
                for (int i4 = 0; i4 < 4; ++i4) {
                  const float4 bb = b4[i4];
                  const float2 s0 = __fadd2_rn(make_float2(v[u][4 * i4 + 0], v[u][4 * i4 + 1]), make_float2(bb.x, bb.y));
                  const float2 s1 = __fadd2_rn(make_float2(v[u][4 * i4 + 2], v[u][4 * i4 + 3]), make_float2(bb.z, bb.w));
                  hv[2 * i4 + 0] = relu_half2(s0);
                  hv[2 * i4 + 1] = relu_half2(s1);
                }
              }
              const int kc = kc0 + gi * 2;
#ifndef P2S_ABL_NOA2
              *reinterpret_cast<uint4*>(dst + kc * 128) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
              *reinterpret_cast<uint4*>(dst + (kc + 1) * 128) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
#else
              if (hv[0] == 12345u) *reinterpret_cast<uint4*>(dst + kc * 128) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
#endif
            }
          }
        }
#ifdef P2S_PROFILE
        const long long td1 = clock64();
#endif
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_SCR_FREE], 0);
#ifdef P2S_PROFILE
        prof_acc[17] += (unsigned long long)(td1 - td0);
        prof_acc[18] += (unsigned long long)(clock64() - td1);
#endif
      }
      { PROF_T0(); WAIT_EPI(&bars[BAR_ACC_FULL], acc_waits & 1); PROF_ADD(15); }
      ++acc_waits;
      if (acc_waits == 1 && warp == kWarpEpi0 && lane == 0) STAMP(7);
      tc_fence_after();
#ifdef P2S_PROFILE
      const long long te0 = clock64();
#endif
      const int x = x0 + m;
      const int GK = p.Nk >> 4;
      const int GF = p.K >> 4, tail = p.K & 15;  // full 16-column groups, real columns after them
      if (pmode == 2) {
        // adjoint: dL/dbeta_k = sum_c dL/dJ_c C_kc, with C_kc = C'_kc + 0.5 s_k
        // (C' convolves the centred image; s_k = tap sum of phi_k)
        const bool st = store && x < p.W;
        const size_t pix = (size_t)y * p.W + x;
        const float* gJb = p.gJ + (size_t)b * C * HW + pix;
        float* ob = p.beta_out + (size_t)b * p.K * HW + pix;
        if (C == 3) adj_epi<3>(tl, p.Nk, p.K, wg, GK, gJb, HW, p.consts + 128, ob, st);
        else if (C == 2) adj_epi<2>(tl, p.Nk, p.K, wg, GK, gJb, HW, p.consts + 128, ob, st);
        else adj_epi<1>(tl, p.Nk, p.K, wg, GK, gJb, HW, p.consts + 128, ob, st);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_TMEM_FREE], 0);
      } else if (pmode == 1) {
        for (int gi = wg; gi < GK; gi += 2) {
          float bv[16];
          tmem_ld16(tl + p.scr_col + gi * 16, bv);
          tmem_ld_wait();
          if (store && x < p.W)
            for (int i = 0; i < 16 && gi * 16 + i < p.K; ++i)
              p.beta_out[((size_t)b * p.K + gi * 16 + i) * HW + (size_t)y * p.W + x] = bv[i] + (p.bias_folded ? 0.f : sB3[gi * 16 + i]);
        }
      } else if (kAdj == 2) {
        const bool st = store && x < p.Ws;  // pitch columns [W, Ws) get zeros
        const size_t pix = (size_t)y * p.W + x;
        const float* gJb = p.gJ + (size_t)b * C * HW + pix;
        float* ob = p.beta_out ? p.beta_out + (size_t)b * p.K * HW + pix : nullptr;
        __half* ub = p.u_out ? p.u_out + (size_t)b * C * p.K * p.H * p.Ws + (size_t)y * p.Ws + x : nullptr;
        const bool real = x < p.W;
        const size_t plane = (size_t)p.H * p.Ws;
        const uint32_t* umb = p.u_maxbits + (size_t)b * C;
        float jc[3] = {0.f, 0.f, 0.f}, bs = 0.f;
        if (C == 3) adj_u_epi<3>(tl, p.scr_col, p.Nk, p.K, wg, GK, gJb, HW, p.consts, p.bias_folded != 0, ob, ub,
                                 umb, plane, st, real, jc, bs);
        else if (C == 2) adj_u_epi<2>(tl, p.scr_col, p.Nk, p.K, wg, GK, gJb, HW, p.consts, p.bias_folded != 0, ob, ub,
                                      umb, plane, st, real, jc, bs);
        else adj_u_epi<1>(tl, p.scr_col, p.Nk, p.K, wg, GK, gJb, HW, p.consts, p.bias_folded != 0, ob, ub, umb, plane,
                          st, real, jc, bs);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_TMEM_FREE], 0);
        if (p.J) {  // the forward blur J as well (dL/dt needs it): the two warpgroups' halves
          float4* red = sRed + (red_i++ & 1) * 128;
          if (wg == 1) red[m] = make_float4(jc[0], jc[1], jc[2], bs);
          named_bar_sync(1, 32 * kNumEpiWarps);
          if (wg == 0 && store && x < p.W) {
            const float4 o = red[m];
            const float bt = bs + o.w;
            const float jt[3] = {jc[0] + o.x, jc[1] + o.y, jc[2] + o.z};
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c < C) p.J[((size_t)b * C + c) * HW + (size_t)y * p.W + x] = fmaf(0.5f, bt, jt[c]);
          }
        }
      } else {
        // packed fp32x2 accumulation: lane .x sums even k, .y odd k (combined after the loop)
        float2 jc2[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float2 bs2 = make_float2(0.f, 0.f);
#ifdef P2S_ABL_EPI0
        for (int gi = wg; gi < 0; gi += 2) {
#else
        for (int gi = wg; gi < GK; gi += 2) {
#endif
          // a tail group with <= 4 real columns (K % 16 in 1..4, e.g. K = 100) reads only those:
          // the columns past K are zero padding (N % 16 == 0)
          if (gi == GF && tail <= 4) conv_epi_group<4>(tl, p.scr_col, p.Nk, gi, C, sB3, sSv, jc2, bs2, p.bias_folded != 0);
          else conv_epi_group<16>(tl, p.scr_col, p.Nk, gi, C, sB3, sSv, jc2, bs2, p.bias_folded != 0);
        }
        float jc[3] = {jc2[0].x + jc2[0].y, jc2[1].x + jc2[1].y, jc2[2].x + jc2[2].y};
        float bs = bs2.x + bs2.y;
        // every TMEM read of this tile is done: release TMEM before combining / storing J (in a
        // sequence, frames before the last release only beta's scratch: the accumulators stay)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[fr == nfr - 1 ? BAR_TMEM_FREE : BAR_SCR_FREE], 0);
        if (acc_waits == 1 && warp == kWarpEpi0 && lane == 0) STAMP(8);
#ifdef P2S_PROFILE
        prof_acc[16] += (unsigned long long)(clock64() - te0);
#endif
        float4* red = sRed + (red_i++ & 1) * 128;
        if (wg == 1) red[m] = make_float4(jc[0], jc[1], jc[2], bs);
        named_bar_sync(1, 32 * kNumEpiWarps);
        if (wg == 0) {
          const float4 o = red[m];
          bs += o.w;
          jc[0] += o.x; jc[1] += o.y; jc[2] += o.z;
          if (store && x < p.W) {
            // sequence mode: frame b + fr, every channel; colour mode (per-channel beta): frame b,
            // channel fr only (the pass of channel fr's Zernike field)
            const int c0 = p.color ? fr : 0, c1 = p.color ? fr + 1 : C;
            float* jo = p.J + (p.color ? ((size_t)b * C + fr) : (size_t)(b + fr) * C) * HW + (size_t)y * p.W + x;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c >= c0 && c < c1) jo[(size_t)(c - c0) * HW] = fmaf(0.5f, bs, jc[c]);
          }
        }
      }
      if (pmode == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&bars[BAR_TMEM_FREE], 0);
      }
    }
    if (warp == kWarpEpi0 && lane == 0) STAMP(9);
  }
#ifdef P2S_PROFILE
  {
    prof_acc[12] = globaltimer_ns();
    prof_acc[19] = (unsigned long long)(clock64() - prof_start);
    int base = -1;
    if (warp == kWarpMma && lane == 0) base = 0;
    else if (warp == kWarpProducer && lane == 0) base = 1;
    else if (builder_index(warp) == 0 && lane == 0) base = 2;
    else if (warp == kWarpEpi0 && lane == 0) base = 3;
    if (p.prof && base >= 0)
      for (int i = 0; i < 20; ++i)
        if (prof_acc[i]) p.prof[((size_t)blockIdx.x * 4 + base) * 20 + i] = prof_acc[i];
  }
#endif
  // dependents (the warp kernel) may launch once every CTA got here; they still wait for this
  // grid's completion (griddepcontrol.wait) before reading J
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- teardown: no CTA leaves while its pair may still touch its shared memory / TMEM
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x == 0) STAMP_CTA(16 + 160);
  if (warp == kWarpMma) tmem_dealloc2<kTmemCols>(tmem);
}

// Step a3: out(y,x) = bilinear J at (y - t1, x - t0), clamp-to-edge; all channels per thread.
// Vectorised warp for W % 4 == 0: four consecutive pixels of a row per thread (float4 tilt
// loads and output stores; the 4 x C gathers per pixel stay scalar). Launched as a programmatic
// dependent of k_fused_p2s: the tilt (independent of J) is loaded before griddepcontrol.wait,
// so its HBM latency and the launch overlap the fused kernel's tail.
// Rows [wy0, wy0 + wny) of every frame (the host path warps row bands as they complete).
__global__ void __launch_bounds__(256) k_tilt_warp4(const float* __restrict__ J, const float* __restrict__ tilt,
                                                    float* __restrict__ out, int B, int C, int H, int W, int wy0,
                                                    int wny) {
  const size_t HW = (size_t)H * W, BW = (size_t)wny * W;
  const size_t nq = (size_t)B * BW / 4;
  const size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  float4 tx = make_float4(0.f, 0.f, 0.f, 0.f), ty = tx;
  size_t b = 0, pix = 0;
  if (q < nq) {
    b = (q * 4) / BW;
    pix = (size_t)wy0 * W + (q * 4 - b * BW);
    if (tilt) {
      tx = __ldg(reinterpret_cast<const float4*>(tilt + (b * 2 + 0) * HW + pix));
      ty = __ldg(reinterpret_cast<const float4*>(tilt + (b * 2 + 1) * HW + pix));
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // J is complete past this point
  if (q >= nq) return;
  const int y = (int)(pix / W), x = (int)(pix - (size_t)y * W);
  const float txs[4] = {tx.x, tx.y, tx.z, tx.w}, tys[4] = {ty.x, ty.y, ty.z, ty.w};
  int o00[4], o01[4], o10[4], o11[4];
  float w00[4], w01[4], w10[4], w11[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float sy = fminf(fmaxf((float)y - tys[e], -1.f), (float)H);
    const float sx = fminf(fmaxf((float)(x + e) - txs[e], -1.f), (float)W);
    const float fy0 = floorf(sy), fx0 = floorf(sx);
    const float fy = sy - fy0, fx = sx - fx0;
    const int y0 = (int)fy0, x0 = (int)fx0;
    const int ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
    const int xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
    o00[e] = ya * W + xa; o01[e] = ya * W + xb; o10[e] = yb * W + xa; o11[e] = yb * W + xb;
    w00[e] = (1.f - fy) * (1.f - fx); w01[e] = (1.f - fy) * fx; w10[e] = fy * (1.f - fx); w11[e] = fy * fx;
  }
  for (int c = 0; c < C; ++c) {
    const float* Jc = J + (b * C + c) * HW;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = w00[e] * __ldg(Jc + o00[e]) + w01[e] * __ldg(Jc + o01[e]) + w10[e] * __ldg(Jc + o10[e]) +
             w11[e] * __ldg(Jc + o11[e]);
    *reinterpret_cast<float4*>(out + (b * C + c) * HW + pix) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

__global__ void __launch_bounds__(256) k_tilt_warp(const float* __restrict__ J, const float* __restrict__ tilt,
                                                   float* __restrict__ out, int B, int C, int H, int W, int wy0,
                                                   int wny) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const size_t HW = (size_t)H * W, BW = (size_t)wny * W;
  const size_t n = (size_t)B * BW;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / BW, pix = (size_t)wy0 * W + (i - b * BW);
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

// Adjoint of the tilt warp (oracle/adjoint.py): per output pixel p, the
// bilinear weights scatter g_c(p) into dL/dJ (atomicAdd, gJ zeroed by the caller) and
// dL/dt(p) = -sum_c g_c(p) d out_c / d s (0 where the coordinate clamp is active).
// gJ != nullptr: scatter dL/dout into dL/dJ (needs no J); gt != nullptr: dL/dt from J's corners
__global__ void __launch_bounds__(256) k_warp_backward(const float* __restrict__ J, const float* __restrict__ tilt,
                                                       const float* __restrict__ g, float* __restrict__ gJ,
                                                       float* __restrict__ gt, int B, int C, int H, int W) {
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
    const float syr = (float)y - ty, sxr = (float)x - tx;
    const float sy = fminf(fmaxf(syr, -1.f), (float)H), sx = fminf(fmaxf(sxr, -1.f), (float)W);
    const float fy0 = floorf(sy), fx0 = floorf(sx);
    const float fy = sy - fy0, fx = sx - fx0;
    const int y0 = (int)fy0, x0 = (int)fx0;
    const int ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
    const int xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
    const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx, w10 = fy * (1.f - fx), w11 = fy * fx;
    float dsx = 0.f, dsy = 0.f;
    for (int c = 0; c < C; ++c) {
      const float gc = __ldg(g + (b * C + c) * HW + pix);
      if (gJ) {
        float* gJc = gJ + (b * C + c) * HW;
        atomicAdd(gJc + (size_t)ya * W + xa, gc * w00);
        atomicAdd(gJc + (size_t)ya * W + xb, gc * w01);
        atomicAdd(gJc + (size_t)yb * W + xa, gc * w10);
        atomicAdd(gJc + (size_t)yb * W + xb, gc * w11);
      }
      if (gt) {
        const float* Jc = J + (b * C + c) * HW;
        const float j00 = __ldg(Jc + (size_t)ya * W + xa), j01 = __ldg(Jc + (size_t)ya * W + xb);
        const float j10 = __ldg(Jc + (size_t)yb * W + xa), j11 = __ldg(Jc + (size_t)yb * W + xb);
        dsx = fmaf(gc, (1.f - fy) * (j01 - j00) + fy * (j11 - j10), dsx);
        dsy = fmaf(gc, (1.f - fx) * (j10 - j00) + fx * (j11 - j01), dsy);
      }
    }
    if (gt) {
      gt[(b * 2 + 0) * HW + pix] = (sxr > -1.f && sxr < (float)W) ? -dsx : 0.f;
      gt[(b * 2 + 1) * HW + pix] = (syr > -1.f && syr < (float)H) ? -dsy : 0.f;
    }
  }
}

}  // namespace p2s
