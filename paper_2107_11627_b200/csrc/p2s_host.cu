// p2s_host.cu — the C ABI of include/p2s.h: validation, asset packing, execution plan and
// launches of the sm_100a kernels in p2s_kernels.cuh. No torch types, no oracle code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "p2s.h"
#include "p2s_kernels.cuh"
#include "p2s_adjoint.cuh"
#include "p2s_mlp_backward.cuh"

using namespace p2s;

namespace {

thread_local std::string g_last_cuda_error;

p2s_status cuda_fail(cudaError_t e, const char* what) {
  g_last_cuda_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? P2S_ERR_OOM : P2S_ERR_CUDA;
}
#define P2S_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

inline int up16(int v) { return (v + 15) / 16 * 16; }

// Tap of the flipped (correlation-form) kernel psi[a][b] = phi[S-1-a][S-1-b]; a < 0: zero slot.
struct Tap { int a, b; };
struct ConvStep { uint32_t off, lbo; Tap tap[16]; };

// Convolution K-step plan. Correlation form of Eq. (5)'s convolutions:
//   C_k(y,x) = sum_{a,b} psi_k[a][b] * I[cY(y - r + a)][cX(x - r + b)],  psi_k = flip(phi_k)
// The reduction over the S*S taps is cut into 16-tap K-steps, each read from one of the
// 8x-expanded image views with an overlapping UMMA descriptor (SBO = 16 B per pixel):
//   V16: rows a in [16g, 16g+16), one column b       (two EY blocks; LBO = block stride)
//   V8 : rows a in [a0, a0+8), columns b, b+1        (one EY block;  LBO = 16 B)
//   H  : one row a, columns b in [16p, 16p+16)       (one EX row;    LBO = 128 B)
struct ConvPlan {
  std::vector<ConvStep> steps;
  std::vector<int> ey_a0, ex_a;
  int npos_y = 0, npos_x = 0, chan_bytes = 0, rr = 0, chan_bytes1 = 0;
  // half-E mode (ehalf): the E views split by tap rows into two halves with their own buffers --
  // half 0 = EY blocks [0, blkA), half 1 = the rest + the EX rows -- so a tile's second half builds
  // while its first is convolved and the next tile's first half while its second is (double
  // buffering at half the shared memory). Steps [0, cut) read half 0, [cut, n) half 1; offsets are
  // relative to their half's buffer and chan_bytes is the larger half's per-channel size.
  int ehalf = 0, blkA = 0, cut = 0;
};

ConvPlan plan_conv(int S, bool halves = false) {
  ConvPlan P;
  const int r = (S - 1) / 2, rr = (r + 3) / 4 * 4, sh = rr - r;  // E entry 0 <-> column x0 - rr
  const int nv16 = S / 16, L = S - 16 * nv16;
  int left = 0;  // 0 none, 1 H rows, 2 V8 block, 3 extra V16 group
  if (L == 0) left = 0;
  else if (L <= 2 && nv16 > 0) left = 1;
  else if (L <= 8) left = 2;
  else left = 3;
  const int ngroups = nv16 + (left == 3 ? 1 : 0);
  for (int g = 0; g < ngroups; ++g) { P.ey_a0.push_back(16 * g); P.ey_a0.push_back(16 * g + 8); }
  if (left == 2) P.ey_a0.push_back(16 * nv16);
  if (left == 1)
    for (int a = 16 * nv16; a < S; ++a) P.ex_a.push_back(a);
  const int nblk = (int)P.ey_a0.size(), nex = (int)P.ex_a.size();
  const int Pairs = ((S + 7) / 8 + 1) / 2;
  P.npos_y = nblk ? (sh + 128 + S + 1 + 3) / 4 * 4 : 0;
  P.npos_x = nex ? (sh + 128 + 16 * Pairs + 3) / 4 * 4 : 0;
  const uint32_t ystride = (uint32_t)P.npos_y * 16, xbase = (uint32_t)nblk * ystride;
  P.chan_bytes = (int)(xbase + (uint32_t)nex * P.npos_x * 16);
  for (int g = 0; g < ngroups; ++g)
    for (int b = 0; b < S; ++b) {
      ConvStep st{(uint32_t)(2 * g) * ystride + (uint32_t)(b + sh) * 16, ystride, {}};
      for (int kk = 0; kk < 16; ++kk) {
        const int a = 16 * g + 8 * (kk / 8) + (kk % 8);
        st.tap[kk] = a < S ? Tap{a, b} : Tap{-1, -1};
      }
      P.steps.push_back(st);
    }
  if (left == 2) {
    const int a0 = 16 * nv16;
    for (int b = 0; b < S; b += 2) {
      ConvStep st{(uint32_t)(nblk - 1) * ystride + (uint32_t)(b + sh) * 16, 16, {}};
      for (int kk = 0; kk < 16; ++kk) {
        const int a = a0 + kk % 8, bb = b + kk / 8;
        st.tap[kk] = (a < S && bb < S) ? Tap{a, bb} : Tap{-1, -1};
      }
      P.steps.push_back(st);
    }
  }
  for (int e = 0; e < nex; ++e)
    for (int pr = 0; pr < Pairs; ++pr) {
      const int b0 = 16 * pr;
      ConvStep st{xbase + (uint32_t)e * P.npos_x * 16 + (uint32_t)(b0 + sh) * 16, 128, {}};
      for (int kk = 0; kk < 16; ++kk)
        st.tap[kk] = (b0 + kk < S) ? Tap{P.ex_a[e], b0 + kk} : Tap{-1, -1};
      P.steps.push_back(st);
    }
  P.rr = rr;
  P.chan_bytes1 = P.chan_bytes;
  if (halves && ngroups >= 2) {
    const int gA = ngroups / 2, blkA = 2 * gA;
    const uint32_t xbase_b = (uint32_t)(nblk - blkA) * ystride;  // EX rows follow half 1's blocks
    P.ehalf = 1;
    P.blkA = blkA;
    P.cut = gA * S;  // the V16 steps of groups [0, gA)
    P.chan_bytes = (int)((uint32_t)blkA * ystride);
    P.chan_bytes1 = (int)(xbase_b + (uint32_t)nex * P.npos_x * 16);
    for (size_t i = (size_t)P.cut; i < P.steps.size(); ++i) {
      ConvStep& st = P.steps[i];
      if (st.off >= xbase) st.off = st.off - xbase + xbase_b;  // H steps (EX rows)
      else st.off -= (uint32_t)blkA * ystride;                 // V16 / V8 steps of half 1's blocks
    }
  }
  return P;
}

// element (row, k) of a packed 16-K slab (LBO = 128, SBO = 256), in fp16 units
inline size_t slab_idx(int n, int kk) { return ((n % 8) * 16 + (n / 8) * 256 + (kk % 8) * 2 + (kk / 8) * 128) / 2; }

constexpr int kSmemLimit = 232448;  // 227 KB opt-in per block on sm_100

}  // namespace

struct p2s_handle {
  int K, S, r, n_in, h1, h2, Nk, K1, N1, N2;
  ConvPlan plan;
  std::vector<Item> items;  // [items_full | items_beta]
  int n_items_full = 0, n_items_beta = 0, n_items_first = 0, n_items_seq = 0, n_items_conv = 0, tab_cap = 0;
  float* d_gJ = nullptr;  // adjoint workspace dL/dJ
  float* d_col_ws = nullptr;  // colour adjoint: per-channel dL/dt and (if needed) dL/dbeta planes
  size_t col_ws_cap = 0;
  size_t gJ_cap = 0;
  // dL/dI (k_adjoint_image): plan, phi table, workspaces beta [B][K][H][W] fp32 and U_T fp16
  int di_R = 0, di_nchunk = 0, di_kg = 0, di_ngroups = 0, di_Nh = 0, di_OW = 0, di_nring = 0, di_smem = 0;
  int di_a_bytes = 0, di_b_bytes = 0, di_off_p = 0, di_off_bar = 0, di_egroups = 1;
  uint8_t* d_dib = nullptr;
  __half* d_ut = nullptr;
  size_t ut_cap = 0;
  uint32_t* d_umax = nullptr;  // [B*C] max |dL/dJ| bits per plane (U's fp16 range scale)
  size_t umax_cap = 0;
  PFN_cuTensorMapEncodeTiled encode = nullptr;
  // dL/dz (k_mlp_backward): resident weight pack and its shared-memory plan (mb_ok = it fits)
  uint8_t* d_mlpb = nullptr;
  int mb_col_b = 0, mb_col_c = 0, mb_off_z = 0;
  bool mf_ok = false;  // k_mlp_forward usable (resident plan, TMEM regions fit)
  int mb_ok = 0, mb_fold = 0, mb_stream = 0, mb_g3 = 1, mb_nring = 0, mb_slot = 0, mb_off_ring = 0, mb_ring_src_off = 0,
      mb_smem = 0, mb_off_w2 = 0, mb_off_w3 = 0, mb_off_bias = 0, mb_wbytes = 0, mb_off_act = 0, mb_off_bar = 0;
  MlpOp ops[kMaxOps];  // [0, n_ops) per-tile ops, then n_fops first-tile whole-layer ops
  int n_ops = 0, n_fops = 0;
  bool bias_folded = false;
  int stage_bytes, nring, smem_bytes, n_ebuf, scr_col;
  int off_ring, off_a1, off_a2, off_hold, off_e, off_tab, off_const, off_red, off_bar, a1_sbo, a2_sbo, hold_sbo;
  int off_anc = 0, anc_cols = 0;
  int l3_hold_ks = 0, hold_k0 = 0;
  std::vector<MmaItem> mma_items;
  int sm_count;
  uint8_t* d_stream = nullptr;
  Item* d_items = nullptr;
  MmaItem* d_mma = nullptr;
  uint32_t* d_steps = nullptr;
  float* d_consts = nullptr;
  float* d_J = nullptr;
  size_t J_cap = 0;
  float *h_img = nullptr, *h_z = nullptr, *h_t = nullptr, *h_out = nullptr;  // device staging (host path)
  float* h_anc = nullptr;  // anchor-grid staging (p2s_render_anchors_host)
  size_t anc_cap = 0;
  size_t stage_px_cap = 0, stage_chw_cap = 0;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  // host path (p2s_render_host): input-copy stream and its events
  cudaStream_t s_in = nullptr;
  cudaEvent_t ev_entry = nullptr, ev_band = nullptr;
  // host path, output side: row bands are warped and copied back on s_out as soon as the J rows
  // they read are rendered (one event per rendered band, one per warped frame)
  cudaStream_t s_out = nullptr;
  std::vector<cudaEvent_t> ev_rend;
  cudaEvent_t ev_warped = nullptr;
  unsigned long long* prof = nullptr;
  CUtensorMap maps[kMaxMaps];
  int n_maps = 0;
  int progressive = 1;
  int cmax = 3;                 // channels the E buffers and the TMEM layout are planned for
  int beta_col = 0;             // TMEM column of beta (L3's output): scr_col, or its own region
  int mlp_ahead = 0;            // 1: a tile's L1 / L2 run ahead of the previous tile's conv epilogue
  int l1_early = 0;             // 1: the first L1 chunk lies past beta and issues before the accumulators free
  p2s_handle* c1 = nullptr;     // a one-channel plan of the same model (C = 1 calls use it)
  p2s_handle* seq = nullptr;    // a half-E plan of the same model (p2s_render_sequence, C > 1, uses it)
};

namespace {

p2s_status ensure_J(p2s_handle* h, size_t n) {
  if (n <= h->J_cap) return P2S_OK;
  P2S_CUDA(cudaDeviceSynchronize());
  if (h->d_J) cudaFree(h->d_J);
  h->d_J = nullptr;
  h->J_cap = 0;
  P2S_CUDA(cudaMalloc(&h->d_J, n * sizeof(float)));
  h->J_cap = n;
  return P2S_OK;
}

// Device staging of the host path (p2s_render_host): image, out [chw], Zernike [px n_in], tilt
// [2 px], plus its input stream and events. Growing synchronises the device.
p2s_status ensure_stage(p2s_handle* h, size_t px, size_t chw) {
  if (px > h->stage_px_cap || chw > h->stage_chw_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->h_img); cudaFree(h->h_z); cudaFree(h->h_t); cudaFree(h->h_out);
    h->h_img = h->h_z = h->h_t = h->h_out = nullptr;
    h->stage_px_cap = h->stage_chw_cap = 0;
    P2S_CUDA(cudaMalloc(&h->h_img, chw * 4));
    P2S_CUDA(cudaMalloc(&h->h_out, chw * 4));
    P2S_CUDA(cudaMalloc(&h->h_z, px * h->n_in * 4));
    P2S_CUDA(cudaMalloc(&h->h_t, px * 2 * 4));
    h->stage_px_cap = px;
    h->stage_chw_cap = chw;
  }
  if (!h->s_in) {
    P2S_CUDA(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    P2S_CUDA(cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming));
    P2S_CUDA(cudaEventCreateWithFlags(&h->ev_band, cudaEventDisableTiming));
  }
  if (!h->s_out) {
    P2S_CUDA(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    P2S_CUDA(cudaEventCreateWithFlags(&h->ev_warped, cudaEventDisableTiming));
  }
  return P2S_OK;
}

// Adjoint workspaces (p2s_backward): dL/dJ [chw] fp32; with dL/dI also U = beta dL/dJ fp16
// [B C K H Ws] and the per-(frame, channel) range exponents. Growing synchronises the device.
p2s_status ensure_adjoint(p2s_handle* h, int B, int C, int H, int W, bool image) {
  const size_t chw = (size_t)B * C * H * W;
  if (chw > h->gJ_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->d_gJ);
    h->d_gJ = nullptr;
    h->gJ_cap = 0;
    P2S_CUDA(cudaMalloc(&h->d_gJ, chw * sizeof(float)));
    h->gJ_cap = chw;
  }
  if (!image) return P2S_OK;
  const size_t nu = (size_t)B * C * h->K * H * (size_t)((W + 7) / 8 * 8);
  if (nu > h->ut_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->d_ut);
    h->d_ut = nullptr;
    h->ut_cap = 0;
    P2S_CUDA(cudaMalloc(&h->d_ut, nu * sizeof(__half)));
    h->ut_cap = nu;
  }
  const size_t nbc = (size_t)B * C;
  if (nbc > h->umax_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->d_umax);
    h->d_umax = nullptr;
    h->umax_cap = 0;
    P2S_CUDA(cudaMalloc(&h->d_umax, nbc * sizeof(uint32_t)));
    h->umax_cap = nbc;
  }
  return P2S_OK;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b) return false;
  const char *pa = (const char*)a, *pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

FusedParams make_params(const p2s_handle* h, int B, int C, int H, int W, int mode) {
  FusedParams p{};
  p.B = B; p.C = C; p.H = H; p.W = W; p.n_in = h->n_in;
  p.nstrips = (W + kTileM - 1) / kTileM;
  p.y0 = 0;
  p.ny = H;
  p.ntiles = B * p.nstrips * H;
  p.mode = mode;
  p.stream = h->d_stream;
  p.items = h->d_items;
  p.n_items_full = h->n_items_full;
  p.n_items_beta = h->n_items_beta;
  p.n_items_first = h->n_items_first;
  p.n_items_seq = h->n_items_seq;
  p.n_items_conv = h->n_items_conv;
  p.nfr = 1;
  p.tab_cap = h->tab_cap;
  p.off_mma = h->off_tab + h->tab_cap * (int)sizeof(Item);
  p.off_steps = p.off_mma + h->tab_cap * (int)sizeof(MmaItem);
  for (int i = 0; i < h->n_ops + h->n_fops; ++i) p.ops[i] = h->ops[i];
  p.n_ops = h->n_ops;
  p.n_fops = h->n_fops;
  p.bias_folded = h->bias_folded ? 1 : 0;
  p.conv_steps = h->d_steps;
  p.nconv = (int)h->plan.steps.size();
  p.consts = h->d_consts;
  p.K = h->K; p.Nk = h->Nk; p.K1 = h->K1; p.N1 = h->N1; p.N2 = h->N2; p.r = h->r; p.rr = h->plan.rr;
  p.n_ey = (int)h->plan.ey_a0.size(); p.n_ex = (int)h->plan.ex_a.size();
  p.npos_y = h->plan.npos_y; p.npos_x = h->plan.npos_x;
  for (int i = 0; i < p.n_ey; ++i) p.ey_a0[i] = h->plan.ey_a0[i];
  for (int i = 0; i < p.n_ex; ++i) p.ex_a[i] = h->plan.ex_a[i];
  p.chan_bytes = h->plan.chan_bytes;
  p.ehalf = h->plan.ehalf;
  p.blkA = h->plan.blkA;
  p.chan_bytes1 = h->plan.chan_bytes1;
  p.n_ebuf = h->n_ebuf;
  p.scr_col = h->beta_col;  // (the kernel reads beta there; MLP ops carry their own columns)
  p.mlp_ahead = h->mlp_ahead;
  p.stage_bytes = h->stage_bytes; p.nring = h->nring;
  p.off_ring = h->off_ring; p.off_a1 = h->off_a1; p.off_a2 = h->off_a2; p.off_e = h->off_e;
  p.off_tab = h->off_tab; p.off_const = h->off_const; p.off_red = h->off_red; p.off_bar = h->off_bar;
  p.off_hold = h->off_hold;
  p.off_anc = h->off_anc;
  p.anc_cols = h->anc_cols;
  p.smem_bytes = h->smem_bytes;
  p.a1_sbo = h->a1_sbo; p.a2_sbo = h->a2_sbo; p.hold_sbo = h->hold_sbo;
  p.l3_hold_ks = h->l3_hold_ks;
  p.hold_k0 = h->hold_k0;
  p.mma_items = h->d_mma;
  p.prof = h->prof;
  for (int i = 0; i < kMaxMaps; ++i) p.maps[i] = h->maps[i];
  p.progressive = h->progressive;
  p.ecmax = h->cmax;
  return p;
}

p2s_status launch_fused(p2s_handle* h, const FusedParams& p, cudaStream_t st) {
  if (p.ntiles == 0) return P2S_OK;
  // persistent grid of CTA pairs (clusters of 2): at most one CTA per SM
  const int npairs = (p.ntiles + 1) / 2;
  const int grid = 2 * std::max(1, std::min(h->sm_count / 2, npairs));
  if (p.mode == 2) k_fused_p2s<false, 1><<<grid, kThreads, h->smem_bytes, st>>>(p);
  else if (p.mode == 3) k_fused_p2s<false, 2><<<grid, kThreads, h->smem_bytes, st>>>(p);
  else if (p.anchors) k_fused_p2s<true><<<grid, kThreads, h->smem_bytes, st>>>(p);
  else k_fused_p2s<false><<<grid, kThreads, h->smem_bytes, st>>>(p);
  P2S_CUDA(cudaPeekAtLastError());
  return P2S_OK;
}

// Tilt warp (step a3), launched as a programmatic dependent of the fused kernel on `st`
// (its launch and tilt loads overlap the fused kernel's tail; it waits for J on the device).
p2s_status launch_warp(const p2s_handle* h, const float* J, const float* tilt, float* out, int B, int C,
                       int H, int W, cudaStream_t st, int wy0 = 0, int wny = -1, bool pdl = true) {
  if (wny < 0) wny = H;
  const size_t npx = (size_t)B * wny * W;
  const bool vec = (W % 4) == 0 && ((uintptr_t)J % 16) == 0 && ((uintptr_t)out % 16) == 0 &&
                   ((uintptr_t)tilt % 16) == 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  if (vec) {
    cfg.gridDim = dim3((unsigned)((npx / 4 + 255) / 256));
    P2S_CUDA(cudaLaunchKernelEx(&cfg, k_tilt_warp4, J, tilt, out, B, C, H, W, wy0, wny));
  } else {
    cfg.gridDim = dim3((unsigned)std::min<size_t>((npx + 255) / 256, (size_t)h->sm_count * 16));
    P2S_CUDA(cudaLaunchKernelEx(&cfg, k_tilt_warp, J, tilt, out, B, C, H, W, wy0, wny));
  }
  return P2S_OK;
}

// Step a1 for B frames by k_mlp_forward (the resident dL/dz plan's weights, offsets and threads)
p2s_status launch_mlp_forward(const p2s_handle* h, const float* z, int B, int H, int W, float* beta,
                              cudaStream_t st) {
  const size_t HW = (size_t)H * W;
  const long long tpf = ((long long)HW + 127) / 128;
  if (tpf * B > 0x7fffffffLL || (unsigned long long)std::max(h->K, h->n_in + 2) * HW > 0x7fffffffULL)
    return P2S_ERR_UNSUPPORTED;
  MlpbParams p{};
  p.z = z; p.wpack = h->d_mlpb; p.b3 = h->d_consts; p.beta = beta;
  p.B = B; p.HW = (int)HW; p.n_in = h->n_in; p.K = h->K;
  p.K1 = h->K1; p.N1 = h->N1; p.N2 = h->N2; p.Nk = h->Nk;
  p.tiles_per_frame = (int)tpf;
  p.ntiles = (int)(tpf * B);
  p.off_w2 = h->mb_off_w2; p.off_w3 = h->mb_off_w3; p.off_bias = h->mb_off_bias; p.wbytes = h->mb_wbytes;
  p.off_act = h->mb_off_act; p.off_bar = h->mb_off_bar;
  p.col_b = h->mb_col_b; p.col_c = h->mb_col_c; p.off_z = h->mb_off_z;
  const int grid = std::min(p.ntiles, h->sm_count);
  if (h->mb_fold) k_mlp_forward<true><<<grid, kMbThreads, h->mb_smem, st>>>(p);
  else k_mlp_forward<false><<<grid, kMbThreads, h->mb_smem, st>>>(p);
  P2S_CUDA(cudaPeekAtLastError());
  return P2S_OK;
}

p2s_status check_image(const p2s_handle* h, const p2s_image& im) {
  if (!h || !im.data) return P2S_ERR_INVALID_ARG;
  if (im.B < 1 || im.H < 1 || im.W < 1 || im.C < 1) return P2S_ERR_INVALID_ARG;
  if (im.C > 3) return P2S_ERR_UNSUPPORTED;
  if ((long long)im.B * im.H * ((im.W + kTileM - 1) / kTileM) > 0x7fffffffLL) return P2S_ERR_UNSUPPORTED;
  return P2S_OK;
}

}  // namespace

extern "C" {

const char* p2s_status_string(p2s_status s) {
  switch (s) {
    case P2S_OK: return "P2S_OK";
    case P2S_ERR_INVALID_ARG: return "P2S_ERR_INVALID_ARG";
    case P2S_ERR_UNSUPPORTED: return "P2S_ERR_UNSUPPORTED";
    case P2S_ERR_CUDA: return "P2S_ERR_CUDA";
    case P2S_ERR_OOM: return "P2S_ERR_OOM";
  }
  return "P2S_ERR_UNKNOWN";
}

const char* p2s_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

}  // extern "C"

namespace {
// The handle for frames of up to `cmax` channels: E buffers for cmax channels, the MLP scratch
// after cmax conv accumulators. cmax = 1 leaves 400 TMEM columns for the MLP, so
// each layer is one op (three MLP round trips per tile instead of five) and the E buffers take a
// third of the shared memory.
// force_half: take the half-E plan (two half buffers, a larger ring) where it exists even if two full
// E buffers fit -- the plan of the sequence sub-handle; *out_handle is then null
// (P2S_OK) when that plan does not exist or the default plan is a half-E plan already.
p2s_status init_impl(const p2s_basis* basis, const p2s_mlp* mlp, int cmax, p2s_handle** out_handle,
                     bool force_half = false) {
  if (!basis || !mlp || !out_handle || !basis->taps || !mlp->W1 || !mlp->b1 || !mlp->W2 ||
      !mlp->b2 || !mlp->W3 || !mlp->b3)
    return P2S_ERR_INVALID_ARG;
  *out_handle = nullptr;
  const int K = basis->K, S = basis->S;
  if (K < 1 || S < 1 || mlp->n_in < 1 || mlp->h1 < 1 || mlp->h2 < 1) return P2S_ERR_INVALID_ARG;
  if (mlp->n_out != K) return P2S_ERR_INVALID_ARG;
  if (S % 2 == 0 || S > 65 || K > 128 || mlp->n_in > 64 || mlp->h1 > 256 || mlp->h2 > 256)
    return P2S_ERR_UNSUPPORTED;
  int dev = 0;
  P2S_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  P2S_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0) {
    g_last_cuda_error = "device is not sm_100";
    return P2S_ERR_UNSUPPORTED;
  }

  p2s_handle* h = new (std::nothrow) p2s_handle();
  if (!h) return P2S_ERR_OOM;
  h->cmax = cmax;
  h->K = K; h->S = S; h->r = (S - 1) / 2;
  h->n_in = mlp->n_in; h->h1 = mlp->h1; h->h2 = mlp->h2;
  h->Nk = up16(K); h->K1 = up16(mlp->n_in); h->N1 = up16(mlp->h1); h->N2 = up16(mlp->h2);
  h->plan = plan_conv(S);
  const ConvPlan plan_half = plan_conv(S, true);  // used when full double-buffered E views do not fit
  h->sm_count = prop.multiProcessorCount;
  if (const char* e = std::getenv("P2S_PROGRESSIVE")) h->progressive = std::atoi(e) != 0;
  const ConvPlan& P = h->plan;
  const int nconv = (int)P.steps.size();
  if (nconv > kMaxConvSteps) { delete h; return P2S_ERR_UNSUPPORTED; }

  // Biases folded into the GEMMs when every layer's input has a padding column to carry a
  // constant 1: the drains are then a single relu-convert per two values.
  h->bias_folded = h->n_in + 2 <= h->K1 && h->h1 + 2 <= h->N1 && h->h2 + 2 <= h->N2;
  if (const char* e = std::getenv("P2S_NO_BIAS_FOLD")) h->bias_folded = std::atoi(e) == 0 && h->bias_folded;

  // ---- TMEM: conv accumulators [0, 3*Nk), MLP scratch / beta [3*Nk, 3*Nk + CH)
  h->scr_col = cmax * h->Nk;
  const int CH = std::min(256, (512 - h->scr_col) / 16 * 16);  // widest MLP chunk
  // ---- MLP ops: each layer split into <= 2 column chunks of <= CH (L3 = one chunk = beta)
  const int layer_N[3] = {h->N1, h->N2, h->Nk};
  const int layer_K[3] = {h->K1, h->N1, h->N2};
  h->n_ops = 0;
  for (int l = 0; l < 3; ++l) {
    const int N = layer_N[l];
    const int nch = (N + CH - 1) / CH;
    if (nch > 2 || (l == 2 && nch > 1)) { delete h; return P2S_ERR_UNSUPPORTED; }
    // columns [0, w0) and [w0, N), w0 = 160 (P2S_MLP_W0 tunes it): the upper chunk is the L2 one
    // parked in the hold buffer, so a wide lower chunk frees shared memory for the ring -- round 2,
    // measured against w0 = 128: cfg3 fused 176.5 -> 174.5 us, cfg5 401-415 -> 467-479 frames/s,
    // cfg2 17.8k -> 18.4k frames/s (176: no better on cfg3, 470 on cfg5)
    int w0 = nch == 1 ? N : std::max(N - CH, std::min(CH, 160));
    if (const char* e = std::getenv("P2S_MLP_W0"))
      if (nch == 2) w0 = std::max(N - CH, std::min(CH, std::atoi(e) / 16 * 16));
    if (nch == 1) {
      h->ops[h->n_ops++] = MlpOp{l, 0, N, layer_K[l] / 16, 1, 1, h->scr_col};
    } else {
      // the upper (narrower) chunk goes first: for L2 it is the one parked in the hold buffer
      // while the lower chunk still reads A2, so the hold buffer is as small as possible
      h->ops[h->n_ops++] = MlpOp{l, w0, N - w0, layer_K[l] / 16, 1, 0, h->scr_col};
      h->ops[h->n_ops++] = MlpOp{l, 0, w0, layer_K[l] / 16, 0, 1, h->scr_col};
    }
  }
  // One-channel plan with every layer a single op: beta gets its own TMEM region after the L1/L2
  // scratch, so the next tile's L1 and L2 (which only need that scratch and A1) can run while this
  // tile's conv epilogue still reads beta and the accumulator ("MLP ahead"; P2S_NO_AHEAD=1 off)
  h->beta_col = h->scr_col;
  // Early L1 (multi-channel plan): the first L1 chunk goes to the columns after beta's, free while
  // the previous tile's epilogue still reads beta and the accumulators, so it issues without
  // waiting for them (the tile's first conv stage waits instead): the tensor core works in the
  // tile-boundary bubble (P2S_NO_L1EARLY=1 off)
  h->l1_early = 0;
  if (h->n_ops >= 2 && h->ops[0].layer == 0 && !h->ops[0].last_of_layer &&
      h->scr_col + h->Nk + h->ops[0].N <= 512 && !std::getenv("P2S_NO_L1EARLY")) {
    h->ops[0].d_col = h->scr_col + h->Nk;
    h->l1_early = 1;
  }
  {
    const int maxN = std::max(h->N1, h->N2);
    if (cmax == 1 && h->n_ops == 3 && h->scr_col + maxN + h->Nk <= 512 && !std::getenv("P2S_NO_AHEAD")) {
      h->beta_col = h->scr_col + maxN;
      h->ops[2].d_col = h->beta_col;
      h->mlp_ahead = 1;
    }
  }
  // (Whole-layer L1/L2 ops for a CTA's first tile, in its still idle accumulator columns, were
  // superseded by building that tile's E views in the epilogue warps and interleaving it like
  // every other tile; the kernel keeps the n_fops hook, unused: n_fops = 0.)
  h->n_fops = 0;

  // The first-issued L2 chunk is parked in a "hold" buffer that L3 reads directly (the other
  // L2 chunk still reads A2); L3 K-steps [hold_k0, hold_k0 + hold_cols/16) come from it.
  int hold_cols = 0, hold_n0 = 0;
  for (int o = 0; o < h->n_ops; ++o)
    if (h->ops[o].layer == 1 && !h->ops[o].last_of_layer) { hold_cols = h->ops[o].N; hold_n0 = h->ops[o].n0; }
  h->l3_hold_ks = hold_cols / 16;
  h->hold_k0 = hold_n0 / 16;

  // ---- shared-memory layout (per CTA; identical in both CTAs of a pair). The item tables are
  //      sized from the number of ring stages, which depends on the stage size: iterate.
  const int a1_bytes = kTileM * h->K1 * 2;
  const int kh = std::max(h->N1, h->N2);
  const int a2_bytes = kTileM * kh * 2;
  const int hold_bytes = kTileM * hold_cols * 2;
  int e1_bytes = cmax * P.chan_bytes;
  int conv_cut = 0;  // half-E plans: conv items never straddle step `cut`
  const int const_bytes = (h->bias_folded ? 256 : 256 + 2 * kMaxN) * 4;  // b1, b2 unused when folded
  const int red_bytes = 2 * 128 * 16;
  // anchor-grid mode: y-interpolated anchor rows of one tile [n_in][kAncCols] (kernel falls back to
  // direct gathers when a 128-px tile spans more anchor columns, e.g. G > ~80 at W = 512)
  constexpr int kAncCols = 20;
  const int anc_bytes = h->n_in * kAncCols * 4;
  auto al = [](int v) { return (v + 127) / 128 * 128; };
  const int bar_bytes = (BAR_RING + 2 * 4) * 8 + 16;  // BAR_RING fixed barriers + ring
  const bool red_in_hold = hold_bytes >= red_bytes;  // the J reduction buffer reuses the hold buffer
  const int max_half_slab = std::max(std::max(h->N1, h->N2), h->Nk) / 2 * 32;
  // number of ring stages of one op / of the conv for stage size sb (mirrors make_items below)
  auto count_stages = [&](int sb, int nks, int N, bool l3) {
    const int per = std::max(1, sb / (N * 16));
    int n = 0;
    for (int s0 = 0; s0 < nks;) {
      int ns = std::min(per, nks - s0);
      if (l3) {
        const int c0 = h->hold_k0, c1 = h->hold_k0 + h->l3_hold_ks;
        if (s0 < c0) ns = std::min(ns, c0 - s0);
        else if (s0 < c1) ns = std::min(ns, c1 - s0);
      }
      s0 += ns;
      ++n;
    }
    return n;
  };
  auto table_need = [&](int sb) {
    int mlp = 0;
    for (int o = 0; o < h->n_ops; ++o)
      mlp += count_stages(sb, h->ops[o].nks, h->ops[o].N, h->ops[o].layer == 2 && h->l3_hold_ks > 0);
    const int conv = conv_cut ? count_stages(sb, conv_cut, h->Nk, false) + count_stages(sb, nconv - conv_cut, h->Nk, false)
                              : count_stages(sb, nconv, h->Nk, false);
    int fst = 0;  // first-tile list: whole-layer L1 / L2 (or the per-tile L1 / L2), L3, conv
    for (int o = 0; o < h->n_ops + h->n_fops; ++o) {
      const bool in_first = h->n_fops > 0 ? (o >= h->n_ops || h->ops[o].layer == 2) : true;
      if (in_first) fst += count_stages(sb, h->ops[o].nks, h->ops[o].N, h->ops[o].layer == 2 && h->l3_hold_ks > 0);
    }
    return std::max(mlp + conv + fst + conv + mlp, 2 * mlp);  // [first | steady | seq] or [beta | beta]
  };
  int tab_cap = 48, sb = 0, nring = 3;
  for (int iter = 0; iter < 6; ++iter) {
    const int tab_all = tab_cap * (int)(sizeof(Item) + sizeof(MmaItem)) + nconv * 4;
    const int fixed = al(a1_bytes) + al(a2_bytes) + al(hold_bytes) + al(tab_all) + al(const_bytes) +
                      (red_in_hold ? 0 : al(red_bytes)) + al(bar_bytes) + al(anc_bytes);
    int ring_avail = 0;
    const int ebuf_max = std::getenv("P2S_NEBUF") ? std::max(1, std::min(2, std::atoi(std::getenv("P2S_NEBUF")))) : 2;
    // E views: two full buffers if they leave >= 3 ring stages of 12 KB; else two half buffers
    // (plan_half, tap rows split in two); else one full buffer (P2S_EHALF = 1 / 0 forces / forbids
    // the half plan where it exists)
    const char* eh_env = std::getenv("P2S_EHALF");
    const int eh_pref = eh_env ? std::atoi(eh_env) : -1;
    const int e1_full = cmax * h->plan.chan_bytes, e2_half = cmax * (plan_half.chan_bytes + plan_half.chan_bytes1);
    const bool full2_fits = kSmemLimit - fixed - al(2 * e1_full) - 1024 >= 3 * 12288;
    const bool use_half = plan_half.ehalf && ebuf_max == 2 &&
                          (force_half || eh_pref == 1 || (eh_pref != 0 && !full2_fits));
    if (force_half && (!plan_half.ehalf || ebuf_max != 2 || !full2_fits || eh_pref >= 0)) {
      delete h;  // no separate half-E plan to make
      return P2S_OK;
    }
    e1_bytes = use_half ? (e2_half + 1) / 2 : e1_full;  // (n_ebuf * e1_bytes covers both halves)
    conv_cut = use_half ? plan_half.cut : 0;
    if (use_half) {
      h->n_ebuf = 2;
      e1_bytes = (e2_half + 1) / 2;
    } else {
      for (h->n_ebuf = ebuf_max; h->n_ebuf >= 1; --h->n_ebuf) {
        ring_avail = kSmemLimit - fixed - al(h->n_ebuf * e1_bytes) - 1024;
        if (ring_avail >= 3 * 12288) break;
      }
      if (h->n_ebuf < 1) h->n_ebuf = 1;
    }
    ring_avail = kSmemLimit - fixed - al(h->n_ebuf * e1_bytes) - 1024;
    // prefer 3 large stages (fewer ring transitions for the UMMA issuer), else 4, else 2
    // (P2S_NRING overrides the stage count for tuning experiments)
    nring = 3;
    if (const char* e = std::getenv("P2S_NRING")) nring = std::max(2, std::min(8, std::atoi(e)));
    sb = std::min(32768, (ring_avail / nring) / 128 * 128);
    if (sb < 16384 && !std::getenv("P2S_NRING")) {
      nring = 4;
      sb = std::min(32768, (ring_avail / 4) / 128 * 128);
      if (sb < 12288) { nring = 2; sb = std::min(32768, (ring_avail / 2) / 128 * 128); }
    }
    if (sb < max_half_slab) { delete h; return P2S_ERR_UNSUPPORTED; }
    const int need = table_need(sb);
    if (need <= tab_cap) break;
    tab_cap = (need + 7) / 8 * 8;
  }
  if (table_need(sb) > tab_cap) { delete h; return P2S_ERR_UNSUPPORTED; }
  if (conv_cut) h->plan = plan_half;  // (P refers to h->plan: same taps, half-relative offsets)
  h->tab_cap = tab_cap;
  h->nring = nring;
  h->stage_bytes = sb;
  int off = 0;
  h->off_ring = off; off += nring * sb;
  h->off_a1 = off; off += al(a1_bytes);
  h->off_a2 = off; off += al(a2_bytes);
  h->off_hold = off; off += al(hold_bytes);
  h->off_e = off; off += al(h->n_ebuf * e1_bytes);
  h->off_tab = off; off += al(tab_cap * (int)(sizeof(Item) + sizeof(MmaItem)) + nconv * 4);
  h->off_const = off; off += al(const_bytes);
  if (red_in_hold) {
    h->off_red = h->off_hold;
  } else {
    h->off_red = off; off += al(red_bytes);
  }
  h->off_anc = off; off += al(anc_bytes);
  h->anc_cols = kAncCols;
  h->off_bar = off; off += (BAR_RING + 2 * nring) * 8 + 16;
  h->smem_bytes = off;
  h->a1_sbo = (h->K1 / 8) * 128;
  h->a2_sbo = (kh / 8) * 128;
  h->hold_sbo = std::max(16, hold_cols / 8 * 128);
  if (h->smem_bytes > kSmemLimit) { delete h; return P2S_ERR_UNSUPPORTED; }

  // ---- pack the streamed B operands: per op, [rank-0 halves of all slabs][rank-1 halves],
  //      then the conv slabs the same way. Half r of slab ks of an op of width N = rows
  //      [r*N/2, (r+1)*N/2) of the chunk, K columns [16ks, 16ks+16), LBO 128 / SBO 256.
  const int n_all_ops = h->n_ops + h->n_fops;
  std::vector<size_t> op_off(n_all_ops);
  size_t total = 0;
  for (int o = 0; o < n_all_ops; ++o) { op_off[o] = total; total += (size_t)h->ops[o].nks * h->ops[o].N * 32; }
  const size_t conv_off = total;
  total += (size_t)nconv * h->Nk * 32;
  std::vector<__half> stream(total / 2, __float2half(0.f));
  auto put = [&](size_t base, int nks, int N, int ks, int n, int kk, float v) {
    const int half = N / 2, r = n / half, nl = n % half;
    const size_t hs = (size_t)half * 32;  // bytes of one half slab
    stream[(base + (size_t)r * nks * hs + (size_t)ks * hs) / 2 + slab_idx(nl, kk)] = __float2half_rn(v);
  };
  const float* Wl[3] = {mlp->W1, mlp->W2, mlp->W3};
  const float* bl[3] = {mlp->b1, mlp->b2, mlp->b3};
  const int outl[3] = {h->h1, h->h2, K}, inl[3] = {h->n_in, h->h1, h->h2};
  for (int o = 0; o < n_all_ops; ++o) {
    const MlpOp& op = h->ops[o];
    const int l = op.layer;
    for (int ks = 0; ks < op.nks; ++ks)
      for (int n = 0; n < op.N; ++n)
        for (int kk = 0; kk < 16; ++kk) {
          const int row = op.n0 + n, k = ks * 16 + kk;
          if (row < outl[l] && k < inl[l]) {
            put(op_off[o], op.nks, op.N, ks, n, kk, Wl[l][(size_t)row * inl[l] + k]);
          } else if (h->bias_folded && (k == inl[l] || k == inl[l] + 1)) {
            // bias folding: input columns inl[l], inl[l]+1 of every layer are constant 1 (the
            // Zernike tile's padding columns; the previous layer's padding units driven to 1)
            // and carry the bias as an fp16 hi/lo pair (hi + lo = b to ~2^-22 relative: b3 is
            // amplified by the tap sums in the centring term, plain fp16 costs accuracy)
            if (row < outl[l]) {
              const float bh = __half2float(__float2half_rn(bl[l][row]));
              put(op_off[o], op.nks, op.N, ks, n, kk, k == inl[l] ? bh : bl[l][row] - bh);
            } else if ((row == outl[l] || row == outl[l] + 1) && l < 2 && k == inl[l]) {
              put(op_off[o], op.nks, op.N, ks, n, kk, 1.f);
            }
          }
        }
  }
  for (int g = 0; g < nconv; ++g)
    for (int n = 0; n < K; ++n)
      for (int kk = 0; kk < 16; ++kk) {
        const Tap t = P.steps[g].tap[kk];
        if (t.a < 0) continue;
        // psi[a][b] = phi[S-1-a][S-1-b]  (true convolution, A2)
        put(conv_off, nconv, h->Nk, g, n, kk, basis->taps[((size_t)n * S + (S - 1 - t.a)) * S + (S - 1 - t.b)]);
      }

  // ---- per-tile-pair item lists (ring stages in issue order)
  // one tensor map per distinct half-slab height (N/16 rows of 256 B)
  std::vector<int> map_rows;
  auto map_of = [&](int N) {
    const int rows = N / 16;
    for (size_t i = 0; i < map_rows.size(); ++i)
      if (map_rows[i] == rows) return (int)i;
    map_rows.push_back(rows);
    return (int)map_rows.size() - 1;
  };
  auto make_items = [&](size_t base, int nks, int N, uint8_t kind, uint8_t op, std::vector<Item>& out) {
    const uint32_t hs = (uint32_t)N * 16, per = std::max<uint32_t>(1, (uint32_t)sb / hs);
    const int mi = map_of(N);
    // L3 items never straddle the hold-buffer / A2 boundary of their A operand; conv items of a
    // half-E plan never straddle its half boundary
    const bool is_l3 = kind == 0 && h->ops[op].layer == 2 && h->l3_hold_ks > 0;
    const int cut0 = h->hold_k0, cut1 = h->hold_k0 + h->l3_hold_ks;
    const int ecut = kind == 1 ? h->plan.cut : 0;
    for (int s0 = 0; s0 < nks;) {
      int ns = std::min<int>(per, nks - s0);
      if (is_l3) {
        if (s0 < cut0) ns = std::min(ns, cut0 - s0);
        else if (s0 < cut1) ns = std::min(ns, cut1 - s0);
      }
      if (ecut > 0 && s0 < ecut) ns = std::min(ns, ecut - s0);
      Item it{};
      it.src_off = (uint32_t)(base + (size_t)s0 * hs);
      it.bytes = (uint32_t)ns * hs;
      it.half_stride = (uint32_t)nks * hs;
      it.first = (uint16_t)s0;
      it.nslabs = (uint16_t)ns;
      it.kind = kind;
      it.op = op;
      it.flags = (s0 == 0 ? IT_BEGIN : 0) | (s0 + ns >= nks ? IT_END : 0);
      it.map = (uint8_t)mi;
      it.rows = (uint8_t)(N / 16);
      out.push_back(it);
      s0 += ns;
    }
  };
  std::vector<Item> conv_items;
  make_items(conv_off, nconv, h->Nk, 1, 0, conv_items);
  std::vector<Item> full, beta;
  // Issue order: L1c0, then MLP ops spread evenly over the conv stages (>= 1 stage between
  // consecutive ops so the epilogue's drain overlaps tensor work); L3 always precedes the
  // last conv stage so the ACC_FULL commit covers beta.
  const int ncs = (int)conv_items.size();
  const int gaps = std::max(1, h->n_ops - 1);
  const int per_gap = std::max(1, (ncs - 1) / gaps);
  size_t ci = 0;
  if (h->mlp_ahead) {
    // MLP ahead: L1, L2 back to back (they do not wait for the accumulators), the conv stages (the
    // first waits for the previous tile's epilogue), L3 after a third of them
    for (int o = 0; o < h->n_ops; ++o) make_items(op_off[o], h->ops[o].nks, h->ops[o].N, 0, (uint8_t)o, beta);
    for (int o = 0; o < 2; ++o) make_items(op_off[o], h->ops[o].nks, h->ops[o].N, 0, (uint8_t)o, full);
    for (int k = 0; k < std::max(1, ncs / 3) && ci + 1 < conv_items.size(); ++k) full.push_back(conv_items[ci++]);
    make_items(op_off[2], h->ops[2].nks, h->ops[2].N, 0, (uint8_t)2, full);
  } else {
    for (int o = 0; o < h->n_ops; ++o) {
      make_items(op_off[o], h->ops[o].nks, h->ops[o].N, 0, (uint8_t)o, full);
      make_items(op_off[o], h->ops[o].nks, h->ops[o].N, 0, (uint8_t)o, beta);
      if (o + 1 < h->n_ops)
        for (int k = 0; k < per_gap && ci + 1 < conv_items.size(); ++k) full.push_back(conv_items[ci++]);
    }
  }
  while (ci < conv_items.size()) full.push_back(conv_items[ci++]);
  // First tile of every CTA: the epilogue warps build its E views up front (they are idle until
  // the first MLP chunk), so it uses the steady interleaved order too (MLP-first, or whole-layer
  // first-tile MLP ops, measured slower: the builders' A1 + E chain of cold loads took ~10 us).
  std::vector<Item> first = full;
  h->n_items_full = (int)full.size();
  h->n_items_beta = (int)beta.size();
  h->n_items_first = (int)first.size();
  h->n_items_seq = (int)beta.size();  // sequence mode: a frame after a tile's first = its MLP ops
  if (h->n_items_full + h->n_items_first + h->n_items_seq > h->tab_cap || 2 * h->n_items_beta > h->tab_cap) {
    delete h;
    return P2S_ERR_UNSUPPORTED;
  }
  h->items = full;
  h->items.insert(h->items.end(), beta.begin(), beta.end());
  h->items.insert(h->items.end(), first.begin(), first.end());
  h->items.insert(h->items.end(), beta.begin(), beta.end());  // seq list (same B stream)
  h->n_items_conv = (int)conv_items.size();  // adjoint (mode 2): conv stages only
  h->items.insert(h->items.end(), conv_items.begin(), conv_items.end());
  // UMMA-side view of every item (precomputed so the issue loop does one LDS.128 per item)
  auto mma_of = [&](const Item& it, int mode, bool first_tile) {
    MmaItem mi{};
    mi.first = it.first;
    mi.nslabs = (uint8_t)it.nslabs;
    if (it.kind == 1) {
      mi.n16 = (uint8_t)(h->Nk / 16);
      // mode 3 = the adjoint's conv-only list: its first stage also waits for the accumulators.
      // Half-E plans: each half's first stage waits for its E buffer, its last releases it.
      const int ecut = h->plan.ehalf ? h->plan.cut : 0, end = it.first + it.nslabs;
      const bool half1 = ecut > 0 && it.first >= ecut;
      const bool e_begin = (it.flags & IT_BEGIN) || (ecut > 0 && it.first == ecut);
      const bool e_end = (it.flags & IT_END) || (ecut > 0 && end == ecut);
      const bool wait_acc = (it.flags & IT_BEGIN) && (mode == 3 || (mode == 0 && (h->mlp_ahead || h->l1_early)));
      mi.flags = MI_CONV | (e_begin ? MI_WAIT_E : 0) | (wait_acc ? MI_WAIT_TMEM : 0) |
                 (e_end ? MI_COMMIT_E : 0) | (half1 ? MI_EHALF1 : 0) | ((it.flags & IT_END) ? MI_COMMIT_ACC : 0);
      return mi;
    }
    const MlpOp& op = h->ops[it.op];
    mi.n16 = (uint8_t)(op.N / 16);
    uint32_t off, sbo;
    if (op.layer == 0) { off = h->off_a1 + it.first * 256; sbo = h->a1_sbo; }
    else if (op.layer == 2 && h->l3_hold_ks > 0 && it.first >= h->hold_k0 && it.first < h->hold_k0 + h->l3_hold_ks &&
             !(first_tile && h->n_fops > 0)) {
      off = h->off_hold + (it.first - h->hold_k0) * 256; sbo = h->hold_sbo;
    } else { off = h->off_a2 + it.first * 256; sbo = h->a2_sbo; }
    mi.a_lo_rel = (off >> 4) | ((128u >> 4) << 16);
    mi.a_hi = (sbo >> 4) | (1u << 14);
    mi.d_col = (uint16_t)op.d_col;
    uint16_t f = 0;
    // mode 2 = a sequence frame after the tile's first: its L1 waits for the previous frame's
    // beta to leave the scratch (SCR_FREE), not for the conv accumulators (they stay)
    if (it.flags & IT_BEGIN) {
      if (op.layer == 0 && op.first_of_layer)
        f |= MI_WAIT_A1 | (mode == 2 ? (h->l1_early ? 0 : MI_WAIT_SCR)
                                     : ((mode == 0 && (h->mlp_ahead || h->l1_early)) ? 0 : MI_WAIT_TMEM));
      else if (mode == 2 && h->l1_early && op.layer == 0 && it.op == 1)
        f |= MI_WAIT_SCR | MI_WAIT_SCR2;  // a sequence frame's L1c1: the previous reduction + L1c0's drain
      else f |= MI_WAIT_SCR;
    }
    if (it.flags & IT_END) {
      if (op.layer == 0 && op.last_of_layer) f |= MI_COMMIT_A1;
      if (op.layer < 2) f |= MI_COMMIT_MLP;
      else if (mode >= 1) f |= MI_COMMIT_ACC;
    }
    mi.flags = f;
    return mi;
  };
  for (const Item& it : full) h->mma_items.push_back(mma_of(it, 0, false));
  for (const Item& it : beta) h->mma_items.push_back(mma_of(it, 1, false));
  for (const Item& it : first) h->mma_items.push_back(mma_of(it, 0, true));
  for (const Item& it : beta) h->mma_items.push_back(mma_of(it, 2, false));
  for (const Item& it : conv_items) h->mma_items.push_back(mma_of(it, 3, false));

  // ---- constants: b3, svec (128 each), b1, b2 (kMaxN each), zero padded;
  //      svec[k] = sum of the taps of phi_k (centred-image identity)
  std::vector<float> consts(2 * kMaxN + 256, 0.f);  // [b3 | svec | b1 | b2]
  for (int i = 0; i < h->h1; ++i) consts[256 + i] = mlp->b1[i];
  for (int i = 0; i < h->h2; ++i) consts[256 + kMaxN + i] = mlp->b2[i];
  for (int i = 0; i < K; ++i) {
    consts[i] = mlp->b3[i];
    double sum = 0.0;
    for (int t = 0; t < S * S; ++t) sum += basis->taps[(size_t)i * S * S + t];
    consts[128 + i] = (float)sum;
  }
  std::vector<uint32_t> steps(nconv);
  for (int g = 0; g < nconv; ++g) steps[g] = (P.steps[g].off >> 4) | ((P.steps[g].lbo >> 4) << 16);

  auto fail = [&](p2s_status st) { p2s_destroy(h); return st; };
  cudaError_t e;
#define UP(dst, src, bytes)                                                                         \
  if ((e = cudaMalloc(&(dst), (bytes))) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc"));   \
  if ((e = cudaMemcpy((dst), (src), (bytes), cudaMemcpyHostToDevice)) != cudaSuccess)               \
    return fail(cuda_fail(e, "cudaMemcpy"));
  UP(h->d_stream, stream.data(), total);
  if ((int)map_rows.size() > kMaxMaps) return fail(P2S_ERR_UNSUPPORTED);
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if ((e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q)) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(cuda_fail(e != cudaSuccess ? e : cudaErrorUnknown, "cuTensorMapEncodeTiled entry point"));
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    h->encode = encode;
    std::memset(h->maps, 0, sizeof(h->maps));
    for (size_t i = 0; i < map_rows.size(); ++i) {
      // the stream viewed as uint8 [total/256][256]; one box = one half slab
      cuuint64_t gdim[2] = {256, (cuuint64_t)(total / 256)};
      cuuint64_t gstride[1] = {256};
      cuuint32_t box[2] = {256, (cuuint32_t)map_rows[i]};
      cuuint32_t estr[2] = {1, 1};
      CUresult cr = encode(&h->maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, h->d_stream, gdim, gstride, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) {
        g_last_cuda_error = "cuTensorMapEncodeTiled failed (" + std::to_string((int)cr) + ")";
        return fail(P2S_ERR_CUDA);
      }
    }
    h->n_maps = (int)map_rows.size();
  }
  UP(h->d_items, h->items.data(), h->items.size() * sizeof(Item));
  UP(h->d_mma, h->mma_items.data(), h->mma_items.size() * sizeof(MmaItem));
  UP(h->d_steps, steps.data(), steps.size() * sizeof(uint32_t));
  UP(h->d_consts, consts.data(), consts.size() * 4);
#undef UP
  if ((e = cudaFuncSetAttribute(k_fused_p2s<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
          cudaSuccess ||
      (e = cudaFuncSetAttribute(k_fused_p2s<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
          cudaSuccess ||
      (e = cudaFuncSetAttribute(k_fused_p2s<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemLimit)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_fused_p2s<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemLimit)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaFuncSetAttribute"));
  {
    // ---- dL/dI plan (p2s_adjoint.cuh): one basis function per ring stage; its U window of
    // nchunk 8-row chunks (even: UMMA K = 16) and N = R x S in two halves of Nh columns
    // R output rows per band share one window of R + S - 1 rows: the R minimising the staged
    // bytes per output row (this CTA's A window + its half of B) such that each half of
    // N = R x S fits one UMMA (<= 256) and >= 3 ring stages fit (measured: the kernel is bound
    // by L2 -> SM delivery, so bytes per output decide)
    // The epilogue runs in up to kDiGroups groups of four warps (each with an S x 128 fp32 P buffer):
    // as many as leave room for the ring (S = 65 takes fewer).
    int R = 0, hr = 0, Nh = 0, wr8 = 0, kg = 1, nchunk = 0, wpad = 0, stage = 0, nring = 0, egroups = 0;
    const int bar_bytes = 256;
    int sp_bytes = 0;
    for (int eg = kDiGroups; eg >= 1 && nring < 3; --eg) {
    sp_bytes = eg * S * 128 * 4;
    const int avail = kSmemLimit - sp_bytes - bar_bytes;
    double best = 1e30;
    egroups = eg;
    for (int Rt = 2; Rt <= 32; Rt += 2) {
      const int Nht = (Rt / 2 * S + 15) / 16 * 16;
      if (Nht > 256) break;
      const int w8 = (S + Rt - 1 + 7) / 8, nch = w8 + (w8 & 1);  // even chunk count: UMMA K = 16
      const int stg = (nch * 2048 + nch * Nht * 16 + 1023) / 1024 * 1024;  // 1 KB: SWIZZLE_128B U tiles
      const int nr = std::min(6, avail / stg);
      if (nr < 3 || nch * 8 > 256) continue;
      const double cost = (double)stg / Rt;
      if (cost < best) {
        best = cost;
        R = Rt; hr = Rt / 2; Nh = Nht; wr8 = w8; nchunk = nch; wpad = nch; stage = stg; nring = nr;
      }
    }
    }
    if (nring < 3) return fail(P2S_ERR_UNSUPPORTED);  // not reached for S <= 65
    {  // every group gets >= 1 output row (an empty group would never release TMEM)
      const int per = (R + egroups - 1) / egroups;
      h->di_egroups = (R + per - 1) / per;
    }
    h->di_R = R; h->di_Nh = Nh; h->di_kg = kg; h->di_nchunk = nchunk; h->di_nring = nring;
    h->di_ngroups = (K + kg - 1) / kg;
    h->di_OW = 128;  // strip stride: strips tile U, partial diagonal sums meet in RED.ADD
    h->di_a_bytes = nchunk * 2048;
    h->di_b_bytes = nchunk * Nh * 16;  // per CTA: two halves x Nh/2 rows
    h->di_off_p = nring * stage;
    h->di_off_bar = h->di_off_p + sp_bytes;
    // >= 120 KB so that one CTA (and one 512-column TMEM allocation) occupies an SM
    h->di_smem = std::max(h->di_off_bar + bar_bytes, 120 * 1024);
    const int cpk = nchunk / kg;  // chunks per basis function (wr8, or wr8 + 1 when padded)
    std::vector<__half> tab((size_t)h->di_ngroups * 2 * h->di_b_bytes / 2, __float2half(0.f));
    for (int g = 0; g < h->di_ngroups; ++g)
      for (int hf = 0; hf < 2; ++hf)
        for (int c = 0; c < nchunk; ++c)
          for (int n = 0; n < Nh; ++n)
            for (int e8 = 0; e8 < 8; ++e8) {
              const int kl = c / cpk, w = (c - kl * cpk) * 8 + e8, k = g * kg + kl;
              const int sr = hf * hr + n / S, j = n % S, i = w - sr;
              if (n >= hr * S || k >= K || i < 0 || i >= S) continue;
              // [g][CTA rho][half][chunk][Nh/2 rows][8]: CTA rho stages rows [rho Nh/2, +Nh/2)
              const int rho = n / (Nh / 2), nl = n % (Nh / 2);
              const size_t at = (((((size_t)g * 2 + rho) * 2 + hf) * nchunk + c) * (Nh / 2) + nl) * 8 + e8;
              tab[at] = __float2half_rn(basis->taps[((size_t)k * S + i) * S + j]);
            }
    if ((e = cudaMalloc(&h->d_dib, tab.size() * sizeof(__half))) != cudaSuccess ||
        (e = cudaMemcpy(h->d_dib, tab.data(), tab.size() * sizeof(__half), cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(cuda_fail(e, "dI table"));
    if ((e = cudaFuncSetAttribute(k_adjoint_image, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
        cudaSuccess)
      return fail(cuda_fail(e, "cudaFuncSetAttribute(k_adjoint_image)"));
    (void)wpad;
  }
  {
    // ---- dL/dz plan (p2s_mlp_backward.cuh). W1 [N1][K1], W2 [N2][N1], W3^T [N2][Nk] as K-major
    // fp16 tiles (+ fp32 biases, or biases folded as hi/lo pairs). Resident variant when the three
    // and one [128][max K] activation tile fit one SM; otherwise (e.g. 33-256-256-100) the
    // streamed variant: two CTAs per SM, every GEMM's weight slabs through a ring from an
    // L2-resident table (P2S_MB_MODE=stream forces it; tests cover both).
    const int K1 = h->K1, N1 = h->N1, N2 = h->N2, Nk = h->Nk;
    const int w1 = N1 * K1 * 2, w2 = N2 * N1 * 2, w3 = N2 * Nk * 2, bb = (N1 + N2) * 4;
    const int kact = std::max(std::max(K1, N1), std::max(N2, Nk));
    const int act_bytes = 128 * kact * 2;
    auto al128 = [](int v) { return (v + 127) / 128 * 128; };
    const int smem_res = al128(w1 + w2 + w3 + bb) + act_bytes + 64 + 4 * 128 * 4;
    // resident variant's TMEM: RA = [0, maxN) (F1, B1), RB = [col_b, +maxN) (F2, B2), RC =
    // [col_c, +K1) (B3; separate so the next tile's F1 overlaps this tile's dL/dz drain)
    const int maxN = std::max(N1, N2);
    const int col_b = maxN + K1 <= 256 ? 256 : maxN, col_c = col_b + maxN;
    const bool res_fits = smem_res <= kSmemLimit && col_c + K1 <= 512 && Nk <= 128;
    // biases as fp16 hi/lo pairs on constant-1 inputs when each layer input has 2 spare columns
    const bool fold = h->n_in + 2 <= K1 && h->h1 + 2 <= N1;
    if (K1 <= 64) {
      // standard K-major tiles: element (n, k) of [rows][kd] at (n%8)*16 + (n/8)*kd*16 + (k%8)*2 + (k/8)*128
      auto at = [](int n, int k, int kd) { return ((n % 8) * 16 + (n / 8) * kd * 16 + (k % 8) * 2 + (k / 8) * 128) / 2; };
      std::vector<__half> W1h((size_t)N1 * K1, __float2half(0.f)), W2h((size_t)N2 * N1, __float2half(0.f)),
          W3h((size_t)N2 * Nk, __float2half(0.f));
      for (int j = 0; j < h->h1; ++j)
        for (int i = 0; i < h->n_in; ++i) W1h[at(j, i, K1)] = __float2half_rn(mlp->W1[(size_t)j * h->n_in + i]);
      for (int j = 0; j < h->h2; ++j)
        for (int i = 0; i < h->h1; ++i) W2h[at(j, i, N1)] = __float2half_rn(mlp->W2[(size_t)j * h->h1 + i]);
      for (int j = 0; j < h->h2; ++j)
        for (int k = 0; k < K; ++k) W3h[at(j, k, Nk)] = __float2half_rn(mlp->W3[(size_t)k * h->h2 + j]);
      if (fold) {
        // z columns n_in, n_in + 1 are 1: W1 carries b1 there as hi + lo; W1 rows h1, h1 + 1 turn
        // them into a1 columns h1, h1 + 1 = 1, where W2 carries b2 as hi + lo
        auto hi = [](float v) { return __float2half_rn(v); };
        auto lo = [](float v) { return __float2half_rn(v - __half2float(__float2half_rn(v))); };
        for (int j = 0; j < h->h1; ++j) {
          W1h[at(j, h->n_in, K1)] = hi(mlp->b1[j]);
          W1h[at(j, h->n_in + 1, K1)] = lo(mlp->b1[j]);
        }
        W1h[at(h->h1, h->n_in, K1)] = __float2half_rn(1.f);
        W1h[at(h->h1 + 1, h->n_in, K1)] = __float2half_rn(1.f);
        for (int j = 0; j < h->h2; ++j) {
          W2h[at(j, h->h1, N1)] = hi(mlp->b2[j]);
          W2h[at(j, h->h1 + 1, N1)] = lo(mlp->b2[j]);
        }
      }
      std::vector<float> bias((size_t)N1 + N2, 0.f);
      for (int j = 0; j < h->h1; ++j) bias[j] = mlp->b1[j];
      for (int j = 0; j < h->h2; ++j) bias[N1 + j] = mlp->b2[j];
      const char* mode = std::getenv("P2S_MB_MODE");
      const bool stream = !res_fits || (mode && std::strcmp(mode, "stream") == 0);
      if (!stream) {
        // resident pack [W1 | W2 | W3^T | b1 | b2], copied to shared memory offset 0
        std::vector<uint8_t> pk((size_t)w1 + w2 + w3 + bb);
        std::memcpy(pk.data(), W1h.data(), w1);
        std::memcpy(pk.data() + w1, W2h.data(), w2);
        std::memcpy(pk.data() + w1 + w2, W3h.data(), w3);
        std::memcpy(pk.data() + w1 + w2 + w3, bias.data(), bb);
        if ((e = cudaMalloc(&h->d_mlpb, pk.size())) != cudaSuccess ||
            (e = cudaMemcpy(h->d_mlpb, pk.data(), pk.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
          return fail(cuda_fail(e, "dz weight pack"));
        if ((e = cudaFuncSetAttribute(k_mlp_backward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_mlp_backward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_mlp_forward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_mlp_forward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess)
          return fail(cuda_fail(e, "cudaFuncSetAttribute(k_mlp_backward)"));
        h->mb_smem = smem_res;
        h->mb_off_w2 = w1;
        h->mb_off_w3 = w1 + w2;
        h->mb_off_bias = w1 + w2 + w3;
        h->mb_wbytes = (int)pk.size();
        h->mb_off_act = al128((int)pk.size());
        h->mb_off_bar = h->mb_off_act + act_bytes;
        h->mb_col_b = col_b;
        h->mb_col_c = col_c;
        // the forward MLP kernel (k_mlp_forward) alternates two regions of max(N1, N2, Nk) columns
        const int wf = std::max(maxN, Nk);
        h->mf_ok = wf <= col_b && col_b + wf <= 512 && !std::getenv("P2S_BETA_FUSED");
        // the z tile's own buffer after s_max, where it fits
        const int off_z = al128(h->mb_off_bar + 64 + 4 * 128 * 4);
        if (std::getenv("P2S_MB_NOZSEP") == nullptr && off_z + 128 * K1 * 2 <= kSmemLimit) {
          h->mb_off_z = off_z;
          h->mb_smem = off_z + 128 * K1 * 2;
        }
      } else {
        // slab table, per tile: [F1: W1 K-slabs | F2: W2 K-slabs | B1: W3^T K-slabs | B2: W2 row
        // pairs (W2^T K'-slabs) | B3: W1 row pairs, g3 per slot]; K-slabs re-laid [N][16]
        // (lbo 128, sbo 256), row pairs as stored (lbo 16 kd, sbo 128)
        // ring depth: as many slots as two CTAs per SM leave room for (a slot refill is an L2 round
        // trip, so the depth sets the slab throughput), at most 16
        const int slot = std::max(std::max(N1, N2), K1) * 32, g3 = std::max(1, slot / (K1 * 32));
        const int per_cta = 233472 / 2 - 1024, fixed = al128(bb) + act_bytes + 288 + 2 * 128 * 4;
        int nring = std::min(16, (per_cta - fixed) / slot);
        if (const char* e = std::getenv("P2S_MB_NRING")) nring = std::max(2, std::min(nring, std::atoi(e)));
        if (nring < 2) return fail(P2S_ERR_UNSUPPORTED);  // not reached inside the envelope
        const int nb3 = N1 / 16;
        const int nsl = K1 / 16 + N1 / 16 + Nk / 16 + N2 / 16 + (nb3 + g3 - 1) / g3;
        std::vector<uint8_t> st((size_t)bb + (size_t)nsl * slot, 0);
        std::memcpy(st.data(), bias.data(), bb);  // [b1 | b2] first
        uint8_t* tab = st.data() + bb;
        int i = 0;
        auto kslab = [&](const std::vector<__half>& Wt, int N, int kd, int ks) {
          __half* d = reinterpret_cast<__half*>(tab + (size_t)i * slot);
          for (int n = 0; n < N; ++n)
            for (int kk = 0; kk < 16; ++kk)
              d[((n % 8) * 16 + (n / 8) * 256 + (kk % 8) * 2 + (kk / 8) * 128) / 2] = Wt[at(n, 16 * ks + kk, kd)];
          ++i;
        };
        for (int ks = 0; ks < K1 / 16; ++ks) kslab(W1h, N1, K1, ks);
        for (int ks = 0; ks < N1 / 16; ++ks) kslab(W2h, N2, N1, ks);
        for (int ks = 0; ks < Nk / 16; ++ks) kslab(W3h, N2, Nk, ks);
        for (int ks = 0; ks < N2 / 16; ++ks, ++i)
          std::memcpy(tab + (size_t)i * slot, reinterpret_cast<const uint8_t*>(W2h.data()) + (size_t)ks * N1 * 32,
                      (size_t)N1 * 32);
        for (int ks = 0; ks < nb3; ks += g3, ++i)
          std::memcpy(tab + (size_t)i * slot, reinterpret_cast<const uint8_t*>(W1h.data()) + (size_t)ks * K1 * 32,
                      (size_t)std::min(g3, nb3 - ks) * K1 * 32);
        const int off_ring = al128(bb), off_act = off_ring + al128(nring * slot), off_bar = off_act + act_bytes;
        const int smem = off_bar + 288 + 2 * 128 * 4;
        if ((e = cudaMalloc(&h->d_mlpb, st.size())) != cudaSuccess ||
            (e = cudaMemcpy(h->d_mlpb, st.data(), st.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
          return fail(cuda_fail(e, "dz slab table"));
        if ((e = cudaFuncSetAttribute(k_mlp_backward_s<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_mlp_backward_s<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
                cudaSuccess)
          return fail(cuda_fail(e, "cudaFuncSetAttribute(k_mlp_backward_s)"));
        h->mb_stream = 1;
        h->mb_smem = smem;
        h->mb_off_bias = 0;
        h->mb_off_ring = off_ring;
        h->mb_off_act = off_act;
        h->mb_off_bar = off_bar;
        h->mb_slot = slot;
        h->mb_g3 = g3;
        h->mb_nring = nring;
        h->mb_ring_src_off = bb;
      }
      h->mb_ok = 1;
      h->mb_fold = fold ? 1 : 0;
    }
  }
  *out_handle = h;
  return P2S_OK;
}

// C = 1 calls run on the one-channel plan when the handle has one
inline p2s_handle* for_c(p2s_handle* h, int C) { return (h && C == 1 && h->c1) ? h->c1 : h; }
}  // namespace

extern "C" {

p2s_status p2s_init(const p2s_basis* basis, const p2s_mlp* mlp, p2s_handle** out_handle) {
  p2s_status s = init_impl(basis, mlp, 3, out_handle);
  if (s != P2S_OK || std::getenv("P2S_NO_C1")) return s;
  p2s_handle* c1 = nullptr;
  const p2s_status s1 = init_impl(basis, mlp, 1, &c1);
  if (s1 == P2S_OK) (*out_handle)->c1 = c1;  // (optional: C = 1 calls fall back to the main plan)
  if (std::getenv("P2S_DEBUG_C1")) std::fprintf(stderr, "p2s: one-channel plan %s\n", p2s_status_string(s1));
  // sequences of multi-channel frames are MLP passes over resident accumulators: the half-E plan's
  // larger ring serves them better; optional, like the one-channel plan
  if (!std::getenv("P2S_NO_SEQPLAN")) {
    p2s_handle* sq = nullptr;
    if (init_impl(basis, mlp, 3, &sq, true) == P2S_OK && sq) (*out_handle)->seq = sq;
  }
  return P2S_OK;
}

p2s_status p2s_reserve(p2s_handle* h, int B, int C, int H, int W) {
  if (!h || B < 1 || C < 1 || H < 1 || W < 1) return P2S_ERR_INVALID_ARG;
  h = for_c(h, C);
  return ensure_J(h, (size_t)B * C * H * W);
}

p2s_status p2s_reserve_ex(p2s_handle* h, int B, int C, int H, int W, unsigned what) {
  if (!h || B < 1 || C < 1 || H < 1 || W < 1 ||
      (what & ~(unsigned)(P2S_RESERVE_RENDER | P2S_RESERVE_HOST | P2S_RESERVE_ADJOINT | P2S_RESERVE_ADJOINT_IMAGE)))
    return P2S_ERR_INVALID_ARG;
  h = for_c(h, C);
  const size_t px = (size_t)B * H * W, chw = px * C;
  p2s_status s = P2S_OK;
  if (what & (P2S_RESERVE_RENDER | P2S_RESERVE_HOST | P2S_RESERVE_ADJOINT | P2S_RESERVE_ADJOINT_IMAGE))
    s = ensure_J(h, chw);
  if (s == P2S_OK && (what & P2S_RESERVE_HOST)) s = ensure_stage(h, px, chw);
  if (s == P2S_OK && (what & (P2S_RESERVE_ADJOINT | P2S_RESERVE_ADJOINT_IMAGE)))
    s = ensure_adjoint(h, B, C, H, W, (what & P2S_RESERVE_ADJOINT_IMAGE) != 0);
  return s;
}

p2s_status p2s_set_profile_events(p2s_handle* h, p2s_event_t ev_begin, p2s_event_t ev_end) {
  if (!h || ((ev_begin == nullptr) != (ev_end == nullptr))) return P2S_ERR_INVALID_ARG;
  h->ev_begin = (cudaEvent_t)ev_begin;
  h->ev_end = (cudaEvent_t)ev_end;
  if (h->c1) p2s_set_profile_events(h->c1, ev_begin, ev_end);
  if (h->seq) p2s_set_profile_events(h->seq, ev_begin, ev_end);
  return P2S_OK;
}

static p2s_status render_impl(p2s_handle* h, p2s_image im, const float* z, const float* tilt, float* out,
                              float* J_out, cudaStream_t st, const float* anchors = nullptr, int G = 0) {
  const size_t n_img = (size_t)im.B * im.C * im.H * im.W;
  const size_t n_z = anchors ? (size_t)im.B * h->n_in * G * G : (size_t)im.B * h->n_in * im.H * im.W;
  if (anchors) z = anchors;  // (aliasing check below covers whichever input is used)
  const size_t n_t = (size_t)im.B * 2 * im.H * im.W;
  float* dst = out ? out : J_out;
  if (overlaps(dst, n_img * 4, im.data, n_img * 4) || overlaps(dst, n_img * 4, z, n_z * 4) ||
      overlaps(dst, n_img * 4, tilt, n_t * 4))
    return P2S_ERR_INVALID_ARG;
  float* J = J_out;
  if (!J) {
    p2s_status s = ensure_J(h, n_img);
    if (s != P2S_OK) return s;
    J = h->d_J;
  }
  FusedParams p = make_params(h, im.B, im.C, im.H, im.W, 0);
  p.image = im.data;
  p.zernike = anchors ? nullptr : z;
  p.anchors = anchors;
  p.G = G;
  p.J = J;
  if (h->ev_begin) P2S_CUDA(cudaEventRecord(h->ev_begin, st));
  p2s_status s = launch_fused(h, p, st);
  if (s != P2S_OK) return s;
  if (h->ev_end) P2S_CUDA(cudaEventRecord(h->ev_end, st));
  if (out) {
    p2s_status sw = launch_warp(h, J, tilt, out, im.B, im.C, im.H, im.W, st);
    if (sw != P2S_OK) return sw;
  }
  return P2S_OK;
}

p2s_status p2s_render(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                      float* out, p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !out) return P2S_ERR_INVALID_ARG;
  return render_impl(h, im, zernike_field, tilt_field, out, nullptr, (cudaStream_t)stream);
}

p2s_status p2s_render_sequence(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                               int F, float* out, p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !out || im.B != 1 || F < 1 || F > 65535) return P2S_ERR_INVALID_ARG;
  const size_t HW = (size_t)im.H * im.W, n_out = (size_t)F * im.C * HW;
  if (overlaps(out, n_out * 4, im.data, (size_t)im.C * HW * 4) ||
      overlaps(out, n_out * 4, zernike_field, (size_t)F * h->n_in * HW * 4) ||
      overlaps(out, n_out * 4, tilt_field, (size_t)F * 2 * HW * 4))
    return P2S_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  s = ensure_J(h, n_out);
  if (s != P2S_OK) return s;
  // the fused pass runs on the sequence sub-plan where there is one (J stays this handle's workspace,
  // so p2s_reserve covers sequences as before)
  p2s_handle* hf = (h->seq && im.C > 1) ? h->seq : h;
  FusedParams p = make_params(hf, 1, im.C, im.H, im.W, 0);
  p.nfr = F;  // tiles of the one image; every tile serves all F frames (J / Zernike frame = fr)
  p.image = im.data;
  p.zernike = zernike_field;
  p.J = h->d_J;
  if (h->ev_begin) P2S_CUDA(cudaEventRecord(h->ev_begin, st));
  s = launch_fused(hf, p, st);
  if (s != P2S_OK) return s;
  if (h->ev_end) P2S_CUDA(cudaEventRecord(h->ev_end, st));
  return launch_warp(h, h->d_J, tilt_field, out, F, im.C, im.H, im.W, st);
}

p2s_status p2s_render_color(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                            float* out, p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !out) return P2S_ERR_INVALID_ARG;
  const size_t HW = (size_t)im.H * im.W, n_out = (size_t)im.B * im.C * HW;
  if (overlaps(out, n_out * 4, im.data, n_out * 4) ||
      overlaps(out, n_out * 4, zernike_field, n_out * h->n_in * 4) ||
      overlaps(out, n_out * 4, tilt_field, (size_t)im.B * 2 * HW * 4))
    return P2S_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  s = ensure_J(h, n_out);
  if (s != P2S_OK) return s;
  if (h->c1 && im.C > 1 && !std::getenv("P2S_COLOR_FUSED")) {
    // channel c of frame b is a one-channel frame with its own field: one launch of the
    // one-channel plan over the B*C frames (image [B*C][1][H][W], fields [B*C][n_in][H][W], J in
    // [B][C][H][W] order), then the warp of the B frames with their shared tilt
    const p2s_image im1{im.data, im.B * im.C, 1, im.H, im.W};
    s = check_image(h->c1, im1);
    if (s != P2S_OK) return s;
    s = render_impl(h->c1, im1, zernike_field, nullptr, nullptr, h->d_J, st);
    if (s != P2S_OK) return s;
    return launch_warp(h, h->d_J, tilt_field, out, im.B, im.C, im.H, im.W, st);
  }
  FusedParams p = make_params(h, im.B, im.C, im.H, im.W, 0);
  p.nfr = im.C;  // per tile: the C channels' convolutions once, then one MLP + J pass per channel
  p.color = 1;
  p.image = im.data;
  p.zernike = zernike_field;
  p.J = h->d_J;
  if (h->ev_begin) P2S_CUDA(cudaEventRecord(h->ev_begin, st));
  s = launch_fused(h, p, st);
  if (s != P2S_OK) return s;
  if (h->ev_end) P2S_CUDA(cudaEventRecord(h->ev_end, st));
  return launch_warp(h, h->d_J, tilt_field, out, im.B, im.C, im.H, im.W, st);
}

p2s_status p2s_backward(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                        const float* grad_out, float* grad_beta, float* grad_tilt, float* grad_image,
                        p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !grad_out || (!grad_beta && !grad_tilt && !grad_image)) return P2S_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t HW = (size_t)im.H * im.W, chw = (size_t)im.B * im.C * HW;
  {  // outputs must not overlap the inputs (or each other)
    const size_t nz = (size_t)im.B * h->n_in * HW * 4, nb = (size_t)im.B * h->K * HW * 4, nt = (size_t)im.B * 2 * HW * 4,
                 ni = chw * 4;
    const void* in[4] = {im.data, zernike_field, tilt_field, grad_out};
    const size_t in_n[4] = {ni, nz, nt, ni};
    const void* outs[3] = {grad_beta, grad_tilt, grad_image};
    const size_t out_n[3] = {nb, nt, ni};
    for (int o = 0; o < 3; ++o) {
      for (int i = 0; i < 4; ++i)
        if (overlaps(outs[o], out_n[o], in[i], in_n[i])) return P2S_ERR_INVALID_ARG;
      for (int o2 = o + 1; o2 < 3; ++o2)
        if (overlaps(outs[o], out_n[o], outs[o2], out_n[o2])) return P2S_ERR_INVALID_ARG;
    }
  }
  s = ensure_J(h, chw);
  if (s != P2S_OK) return s;
  s = ensure_adjoint(h, im.B, im.C, im.H, im.W, grad_image != nullptr);
  if (s != P2S_OK) return s;
  // dL/dJ: dL/dout scattered through the warp's bilinear weights (needs no J)
  P2S_CUDA(cudaMemsetAsync(h->d_gJ, 0, chw * sizeof(float), st));
  const size_t npx = (size_t)im.B * HW;
  const int grid = (int)std::min<size_t>((npx + 255) / 256, (size_t)h->sm_count * 16);
  k_warp_backward<<<grid, 256, 0, st>>>(nullptr, tilt_field, grad_out, h->d_gJ, nullptr, im.B, im.C, im.H, im.W);
  P2S_CUDA(cudaPeekAtLastError());
  const int Ws = (im.W + 7) / 8 * 8;
  if (grad_image) {
    const size_t nbc = (size_t)im.B * im.C;
    // per-(frame, channel) max |dL/dJ|: U = beta dL/dJ is stored in fp16 scaled by a power of two
    // chosen from it, and k_adjoint_image scales its sums back (any finite dL/dout range)
    P2S_CUDA(cudaMemsetAsync(h->d_umax, 0, nbc * sizeof(uint32_t), st));
    const unsigned bpp = (unsigned)std::max<size_t>(1, std::min<size_t>((HW + 4095) / 4096,
                                                                        (size_t)(4 * h->sm_count + nbc - 1) / nbc));
    k_absmax_planes<<<dim3(bpp, (unsigned)nbc), 256, 0, st>>>(h->d_gJ, HW, h->d_umax);
    P2S_CUDA(cudaPeekAtLastError());
  }
  {
    // one pass over the K convolutions: dL/dbeta_k = sum_c dL/dJ_c C_kc; with dL/dt or dL/dI the
    // render flow (MLP + convolutions, kAdj = 2) whose epilogue also forms J and U = beta dL/dJ
    const bool full = grad_tilt || grad_image;
    FusedParams p = make_params(h, im.B, im.C, im.H, im.W, full ? 3 : 2);
    p.image = im.data;
    p.zernike = zernike_field;
    p.gJ = h->d_gJ;
    p.beta_out = grad_beta;
    p.u_out = grad_image ? h->d_ut : nullptr;
    p.u_maxbits = grad_image ? h->d_umax : nullptr;
    p.J = grad_tilt ? h->d_J : nullptr;
    p.Ws = Ws;
    s = launch_fused(h, p, st);
    if (s != P2S_OK) return s;
  }
  if (grad_tilt) {  // dL/dt from J's bilinear corners
    k_warp_backward<<<grid, 256, 0, st>>>(h->d_J, tilt_field, grad_out, nullptr, grad_tilt, im.B, im.C, im.H, im.W);
    P2S_CUDA(cudaPeekAtLastError());
  }
  if (grad_image) {  // dL/dI: the transpose convolution on the tensor cores (k_adjoint_image)
    P2S_CUDA(cudaMemsetAsync(grad_image, 0, chw * sizeof(float), st));
    DiParams d{};
    {
      // U [planes][H][Ws] fp16; box = 64 columns (128 B) x the window's rows x 1 plane, 128B swizzle
      cuuint64_t gdim[3] = {(cuuint64_t)Ws, (cuuint64_t)im.H, (cuuint64_t)im.B * im.C * h->K};
      cuuint64_t gstride[2] = {(cuuint64_t)Ws * 2, (cuuint64_t)im.H * Ws * 2};
      cuuint32_t box[3] = {64, (cuuint32_t)h->di_nchunk * 8, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      CUresult cr = h->encode(&d.umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, h->d_ut, gdim, gstride, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) {
        g_last_cuda_error = "cuTensorMapEncodeTiled (U) failed (" + std::to_string((int)cr) + ")";
        return P2S_ERR_CUDA;
      }
    }
    {
      const cuuint64_t rows = (cuuint64_t)h->di_ngroups * 2 * h->di_b_bytes / 256;
      cuuint64_t gdim[2] = {256, rows};
      cuuint64_t gstride[1] = {256};
      cuuint32_t box[2] = {256, (cuuint32_t)(h->di_b_bytes / 256)};
      cuuint32_t estr[2] = {1, 1};
      CUresult cr = h->encode(&d.bmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, h->d_dib, gdim, gstride, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) {
        g_last_cuda_error = "cuTensorMapEncodeTiled (dI table) failed (" + std::to_string((int)cr) + ")";
        return P2S_ERR_CUDA;
      }
    }
    d.gI = grad_image;
    d.u_maxbits = h->d_umax;
    d.BC = im.B * im.C; d.K = h->K; d.H = im.H; d.W = im.W; d.S = h->S; d.r = h->r;
    d.R = h->di_R; d.nchunk = h->di_nchunk; d.kg = h->di_kg; d.ngroups = h->di_ngroups; d.Nh = h->di_Nh;
    d.OW = h->di_OW;
    d.xs0 = 0;  // strip 0 = U columns [0, 128); its outputs start at -r
    d.nbands = (im.H + 2 * h->r + d.R - 1) / d.R;
    d.nstrips = (im.W - d.xs0 + d.OW - 1) / d.OW;
    d.npairs = (d.nstrips + 1) / 2;
    d.ntiles = d.BC * d.nbands * d.npairs;
    d.a_bytes = h->di_a_bytes; d.b_bytes = h->di_b_bytes; d.nring = h->di_nring;
    d.stage_bytes = (h->di_a_bytes + h->di_b_bytes + 1023) / 1024 * 1024;
    d.off_p = h->di_off_p; d.off_bar = h->di_off_bar;
    d.egroups = h->di_egroups;
    k_adjoint_image<<<2 * std::min(d.ntiles, h->sm_count / 2), 64 + 128 * d.egroups, h->di_smem, st>>>(d);
    P2S_CUDA(cudaPeekAtLastError());
  }
  return P2S_OK;
}

p2s_status p2s_mlp_backward(p2s_handle* h, const float* zernike_field, const float* grad_beta, int B, int H, int W,
                            float* grad_zernike, p2s_stream_t stream) {
  if (!h || !zernike_field || !grad_beta || !grad_zernike || B < 1 || H < 1 || W < 1) return P2S_ERR_INVALID_ARG;
  const size_t HW = (size_t)H * W, nz = (size_t)B * h->n_in * HW, nb = (size_t)B * h->K * HW;
  if (overlaps(grad_zernike, nz * 4, zernike_field, nz * 4) || overlaps(grad_zernike, nz * 4, grad_beta, nb * 4))
    return P2S_ERR_INVALID_ARG;
  if (!h->mb_ok) return P2S_ERR_UNSUPPORTED;
  const long long tpf = ((long long)HW + 127) / 128;
  // the kernel addresses a frame's channels by 32-bit offsets
  if (tpf * B > 0x7fffffffLL || (unsigned long long)std::max(h->K, h->n_in + 2) * HW > 0x7fffffffULL)
    return P2S_ERR_UNSUPPORTED;
  MlpbParams p{};
  p.z = zernike_field; p.gb = grad_beta; p.gz = grad_zernike; p.wpack = h->d_mlpb;
  p.B = B; p.HW = (int)HW; p.n_in = h->n_in; p.K = h->K;
  p.K1 = h->K1; p.N1 = h->N1; p.N2 = h->N2; p.Nk = h->Nk;
  p.tiles_per_frame = (int)tpf;
  p.ntiles = (int)(tpf * B);
  p.off_w2 = h->mb_off_w2; p.off_w3 = h->mb_off_w3; p.off_bias = h->mb_off_bias; p.wbytes = h->mb_wbytes;
  p.off_act = h->mb_off_act; p.off_bar = h->mb_off_bar;
  p.col_b = h->mb_col_b; p.col_c = h->mb_col_c; p.off_z = h->mb_off_z;
  cudaStream_t st = (cudaStream_t)stream;
  if (h->mb_stream) {
    p.ring_src = h->d_mlpb + h->mb_ring_src_off;
    p.off_ring = h->mb_off_ring; p.nring = h->mb_nring; p.slab_stride = h->mb_slot; p.g3 = h->mb_g3;
    const int grid = std::min(p.ntiles, 2 * h->sm_count);  // two CTAs per SM
    if (h->mb_fold) k_mlp_backward_s<true><<<grid, kMbsThreads, h->mb_smem, st>>>(p);
    else k_mlp_backward_s<false><<<grid, kMbsThreads, h->mb_smem, st>>>(p);
  } else {
    const int grid = std::min(p.ntiles, h->sm_count);
    if (h->mb_fold) k_mlp_backward<true><<<grid, kMbThreads, h->mb_smem, st>>>(p);
    else k_mlp_backward<false><<<grid, kMbThreads, h->mb_smem, st>>>(p);
  }
  P2S_CUDA(cudaPeekAtLastError());
  return P2S_OK;
}

}  // extern "C"

namespace {
// grad_tilt[b] = sum_c part[b C + c] over planes of n floats (the colour adjoint's dL/dt)
__global__ void __launch_bounds__(256) k_sum_channels(float* __restrict__ dst, const float* __restrict__ part, int B,
                                                      int C, size_t n) {
  const size_t tot = (size_t)B * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / n, e = i - b * n;
    float acc = 0.f;
    for (int c = 0; c < C; ++c) acc += part[((size_t)b * C + c) * n + e];
    dst[i] = acc;
  }
}
}  // namespace

extern "C" {

p2s_status p2s_backward_color(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                              const float* grad_out, float* grad_beta, float* grad_tilt, float* grad_image,
                              float* grad_zernike, p2s_stream_t stream) {
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !grad_out || (!grad_beta && !grad_tilt && !grad_image && !grad_zernike))
    return P2S_ERR_INVALID_ARG;
  if (grad_zernike && !h->mb_ok) return P2S_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const int B = im.B, C = im.C, H = im.H, W = im.W, K = h->K;
  const size_t HW = (size_t)H * W, BC = (size_t)B * C;
  // Channel c of frame b is a one-channel render with its own beta, and the
  // colour layouts are exactly B*C one-channel frames: image [B][C][H][W] = [BC][1][H][W], fields
  // [B][C][n_in][H][W] = [BC][n_in][H][W], dL/dbeta [BC][K][H][W]. So the adjoint is ONE
  // p2s_backward over BC frames (the tilt replicated per channel), dL/dt summed over the channels
  // afterwards, and one p2s_mlp_backward. Workspace: the replicated tilt and per-channel dL/dt
  // [BC][2][H][W], and dL/dbeta [BC][K][H][W] when only dL/dz is wanted (grown on first use).
  const size_t n_t = tilt_field ? BC * 2 * HW : 0, n_gt = grad_tilt ? BC * 2 * HW : 0;
  const size_t n_gb = (grad_zernike && !grad_beta) ? BC * K * HW : 0;
  const size_t need = n_t + n_gt + n_gb;
  if (need > h->col_ws_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->d_col_ws);
    h->d_col_ws = nullptr;
    h->col_ws_cap = 0;
    P2S_CUDA(cudaMalloc(&h->d_col_ws, need * sizeof(float)));
    h->col_ws_cap = need;
  }
  float* t_rep = tilt_field ? h->d_col_ws : nullptr;
  float* gt_rep = grad_tilt ? h->d_col_ws + n_t : nullptr;
  float* gb = grad_beta ? grad_beta : (n_gb ? h->d_col_ws + n_t + n_gt : nullptr);
  if (tilt_field)
    for (size_t bc = 0; bc < BC; ++bc)
      P2S_CUDA(cudaMemcpyAsync(t_rep + bc * 2 * HW, tilt_field + bc / C * 2 * HW, 2 * HW * sizeof(float),
                               cudaMemcpyDeviceToDevice, st));
  p2s_image one{im.data, (int)BC, 1, H, W};
  if (gb || gt_rep || grad_image) {
    s = p2s_backward(h, one, zernike_field, t_rep, grad_out, gb, gt_rep, grad_image, stream);
    if (s != P2S_OK) return s;
  }
  if (grad_tilt) {
    k_sum_channels<<<(int)std::min<size_t>(((size_t)B * 2 * HW + 255) / 256, (size_t)h->sm_count * 8), 256, 0, st>>>(
        grad_tilt, gt_rep, B, C, 2 * HW);
    P2S_CUDA(cudaPeekAtLastError());
  }
  if (grad_zernike) {
    s = p2s_mlp_backward(h, zernike_field, gb, (int)BC, H, W, grad_zernike, stream);
    if (s != P2S_OK) return s;
  }
  return P2S_OK;
}

p2s_status p2s_render_anchors(p2s_handle* h, p2s_image im, const float* anchors, int G,
                              const float* tilt_field, float* out, p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!anchors || !out || G < 1 || G > 4096) return P2S_ERR_INVALID_ARG;
  return render_impl(h, im, nullptr, tilt_field, out, nullptr, (cudaStream_t)stream, anchors, G);
}

p2s_status p2s_debug_blur_anchors(p2s_handle* h, p2s_image im, const float* anchors, int G, float* J_out,
                                  p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!anchors || !J_out || G < 1 || G > 4096) return P2S_ERR_INVALID_ARG;
  return render_impl(h, im, nullptr, nullptr, nullptr, J_out, (cudaStream_t)stream, anchors, G);
}

p2s_status p2s_debug_blur(p2s_handle* h, p2s_image im, const float* zernike_field, float* J_out,
                          p2s_stream_t stream) {
  h = for_c(h, im.C);
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !J_out) return P2S_ERR_INVALID_ARG;
  return render_impl(h, im, zernike_field, nullptr, nullptr, J_out, (cudaStream_t)stream);
}

p2s_status p2s_debug_beta(p2s_handle* h, const float* zernike_field, int B, int H, int W, float* beta_out,
                          p2s_stream_t stream) {
  if (!h || !zernike_field || !beta_out || B < 1 || H < 1 || W < 1) return P2S_ERR_INVALID_ARG;
  const size_t n_b = (size_t)B * h->K * H * W, n_z = (size_t)B * h->n_in * H * W;
  if (overlaps(beta_out, n_b * 4, zernike_field, n_z * 4)) return P2S_ERR_INVALID_ARG;
  if (h->mf_ok) return launch_mlp_forward(h, zernike_field, B, H, W, beta_out, (cudaStream_t)stream);
  FusedParams p = make_params(h, B, 1, H, W, 1);
  p.zernike = zernike_field;
  p.beta_out = beta_out;
  return launch_fused(h, p, (cudaStream_t)stream);
}

p2s_status p2s_render_host(p2s_handle* h, const float* image_host, int B, int C, int H, int W,
                           const float* zernike_host, const float* tilt_host, float* out_host,
                           p2s_stream_t stream) {
  h = for_c(h, C);
  if (!h || !image_host || !zernike_host || !out_host) return P2S_ERR_INVALID_ARG;
  p2s_image im{nullptr, B, C, H, W};
  im.data = image_host;  // validated below against the device copy
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t HW = (size_t)H * W, px = (size_t)B * HW, chw = px * C;
  s = ensure_stage(h, px, chw);
  if (s != P2S_OK) return s;
  s = ensure_J(h, chw);
  if (s != P2S_OK) return s;
  // Pipelined over row bands (inputs are PCIe-bound): the input stream copies
  // each frame's image and tilt, then its Zernike field band by band (one 2D copy over the
  // n_in planes per band); the caller's stream renders each band as soon as it has landed,
  // then warps the frame and copies it back. The last band is small, so little work is left
  // once the last input byte has arrived. Stream order on `st` is preserved (the input stream
  // starts behind it).
  // P2S_HOST_TRACE=1: print a per-call timeline of the pipeline (development aid)
  static const bool trace = std::getenv("P2S_HOST_TRACE") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> tev;
  auto mark = [&](const char* what, cudaStream_t on) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, on);
    tev.emplace_back(what, e);
  };
  mark("entry", st);
  P2S_CUDA(cudaEventRecord(h->ev_entry, st));
  P2S_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_entry, 0));
  // Band heights: the tail shrinks geometrically (16, 32, 64, 128 rows from the bottom) so each
  // band renders faster than the next one copies (a row of n_in fp32 Zernike planes takes ~3.6x
  // longer over PCIe than to render); the head is split into bands of <= 160 rows.
  std::vector<int> bands;
  {
    std::vector<int> tailb;
    int left = H;
    for (int t = 16; t <= 128 && left > 0; t *= 2) { const int n = std::min(t, left); tailb.push_back(n); left -= n; }
    const int nhead = (left + 159) / 160;
    for (int k = 0; k < nhead; ++k) bands.push_back(left * (k + 1) / nhead - left * k / nhead);
    bands.insert(bands.end(), tailb.rbegin(), tailb.rend());
  }
  while (h->ev_rend.size() < bands.size()) {
    cudaEvent_t e;
    P2S_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->ev_rend.push_back(e);
  }
  std::vector<int> band_y0(bands.size() + 1, 0);
  for (size_t k = 0; k < bands.size(); ++k) band_y0[k + 1] = band_y0[k] + bands[k];
  for (int f = 0; f < B; ++f) {
    const size_t fo_img = (size_t)f * C * HW, fo_z = (size_t)f * h->n_in * HW, fo_t = (size_t)f * 2 * HW;
    P2S_CUDA(cudaMemcpyAsync(h->h_img + fo_img, image_host + fo_img, (size_t)C * HW * 4, cudaMemcpyHostToDevice, h->s_in));
    if (tilt_host)
      P2S_CUDA(cudaMemcpyAsync(h->h_t + fo_t, tilt_host + fo_t, 2 * HW * 4, cudaMemcpyHostToDevice, h->s_in));
    mark("image+tilt in", h->s_in);
    // J is one buffer: the previous frame's warps must have read it before this frame renders
    if (f > 0) P2S_CUDA(cudaStreamWaitEvent(st, h->ev_warped, 0));
    for (size_t k = 0, y0 = 0; k < bands.size(); ++k) {
      const int ny = bands[k];
      if (ny == 0) continue;
      P2S_CUDA(cudaMemcpy2DAsync(h->h_z + fo_z + (size_t)y0 * W, HW * 4, zernike_host + fo_z + (size_t)y0 * W,
                                 HW * 4, (size_t)ny * W * 4, h->n_in, cudaMemcpyHostToDevice, h->s_in));
      mark("zernike band in", h->s_in);
      P2S_CUDA(cudaEventRecord(h->ev_band, h->s_in));
      P2S_CUDA(cudaStreamWaitEvent(st, h->ev_band, 0));
      FusedParams p = make_params(h, 1, C, H, W, 0);
      p.y0 = y0;
      p.ny = ny;
      p.ntiles = p.nstrips * ny;
      p.image = h->h_img + fo_img;
      p.zernike = h->h_z + fo_z;
      p.J = h->d_J;
      s = launch_fused(h, p, st);
      if (s != P2S_OK) return s;
      mark("band rendered", st);
      P2S_CUDA(cudaEventRecord(h->ev_rend[k], st));
      y0 += ny;
    }
    // Output side, band by band on s_out: the warp of rows [a, b) reads J rows within the frame's
    // largest |y tilt| (+2 for the bilinear cell and the clamp) of them, so it waits for the band
    // holding row b - 1 + reach; then those rows go back to the host. Only the last bands' warps
    // and copies are left once the last input band has rendered.
    static const bool one_warp = std::getenv("P2S_HOST_ONEWARP") != nullptr;  // (A/B: the old tail)
    if (one_warp) {
      s = launch_warp(h, h->d_J, tilt_host ? h->h_t + fo_t : nullptr, h->h_out + fo_img, 1, C, H, W, st);
      if (s != P2S_OK) return s;
      P2S_CUDA(cudaMemcpyAsync(out_host + fo_img, h->h_out + fo_img, (size_t)C * HW * 4, cudaMemcpyDeviceToHost, st));
      P2S_CUDA(cudaEventRecord(h->ev_warped, st));
      continue;
    }
    int reach = 2;
    if (tilt_host) {
      const float* ty = tilt_host + fo_t + HW;
      float m = 0.f;
      for (size_t i = 0; i < HW; ++i) m = std::max(m, std::fabs(ty[i]));
      reach = (std::isfinite(m) && m < (float)H) ? (int)std::ceil(m) + 2 : H;
    }
    int waited = -1;
    for (size_t k = 0; k < bands.size(); ++k) {
      const int a = band_y0[k], ny = bands[k];
      if (ny == 0) continue;
      const int need = std::min(H - 1, a + ny - 1 + reach);
      int j = (int)k;
      while (band_y0[j + 1] <= need) ++j;  // the band holding row `need`
      if (j > waited) {
        P2S_CUDA(cudaStreamWaitEvent(h->s_out, h->ev_rend[j], 0));
        waited = j;
      }
      s = launch_warp(h, h->d_J, tilt_host ? h->h_t + fo_t : nullptr, h->h_out + fo_img, 1, C, H, W, h->s_out, a,
                      ny, false);
      if (s != P2S_OK) return s;
      P2S_CUDA(cudaMemcpy2DAsync(out_host + fo_img + (size_t)a * W, HW * 4, h->h_out + fo_img + (size_t)a * W, HW * 4,
                                 (size_t)ny * W * 4, C, cudaMemcpyDeviceToHost, h->s_out));
    }
    mark("out copied", h->s_out);
    P2S_CUDA(cudaEventRecord(h->ev_warped, h->s_out));
  }
  P2S_CUDA(cudaStreamSynchronize(h->s_out));
  P2S_CUDA(cudaStreamSynchronize(st));
  if (trace) {
    cudaDeviceSynchronize();
    for (auto& te : tev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0].second, te.second);
      std::fprintf(stderr, "[p2s host] %8.1f us  %s\n", ms * 1e3f, te.first);
    }
    for (auto& te : tev) cudaEventDestroy(te.second);
    (void)cudaGetLastError();
  }
  return P2S_OK;
}

p2s_status p2s_render_anchors_host(p2s_handle* h, const float* image_host, int B, int C, int H, int W,
                                   const float* anchors_host, int G, const float* tilt_host, float* out_host,
                                   p2s_stream_t stream) {
  h = for_c(h, C);
  if (!h || !image_host || !anchors_host || !out_host || G < 1 || G > 4096) return P2S_ERR_INVALID_ARG;
  p2s_image im{image_host, B, C, H, W};
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t HW = (size_t)H * W, px = (size_t)B * HW, chw = px * C, nanc = (size_t)h->n_in * G * G;
  s = ensure_stage(h, px, chw);
  if (s != P2S_OK) return s;
  if ((size_t)B * nanc > h->anc_cap) {
    P2S_CUDA(cudaDeviceSynchronize());
    cudaFree(h->h_anc);
    h->h_anc = nullptr;
    h->anc_cap = 0;
    P2S_CUDA(cudaMalloc(&h->h_anc, (size_t)B * nanc * 4));
    h->anc_cap = (size_t)B * nanc;
  }
  s = ensure_J(h, chw);
  if (s != P2S_OK) return s;
  // Anchor-grid inputs are small (43 -> ~5 MB per 512^2 RGB frame): per frame the
  // input stream copies image + anchors, the caller's stream renders the frame as soon as they
  // land while the tilt copies behind them, then warps and copies the frame back.
  P2S_CUDA(cudaEventRecord(h->ev_entry, st));
  P2S_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_entry, 0));
  for (int f = 0; f < B; ++f) {
    const size_t fo_img = (size_t)f * C * HW, fo_t = (size_t)f * 2 * HW, fo_a = (size_t)f * nanc;
    P2S_CUDA(cudaMemcpyAsync(h->h_img + fo_img, image_host + fo_img, (size_t)C * HW * 4, cudaMemcpyHostToDevice, h->s_in));
    P2S_CUDA(cudaMemcpyAsync(h->h_anc + fo_a, anchors_host + fo_a, nanc * 4, cudaMemcpyHostToDevice, h->s_in));
    P2S_CUDA(cudaEventRecord(h->ev_band, h->s_in));
    P2S_CUDA(cudaStreamWaitEvent(st, h->ev_band, 0));
    FusedParams p = make_params(h, 1, C, H, W, 0);
    p.image = h->h_img + fo_img;
    p.zernike = nullptr;
    p.anchors = h->h_anc + fo_a;
    p.G = G;
    p.J = h->d_J;
    s = launch_fused(h, p, st);
    if (s != P2S_OK) return s;
    if (tilt_host) {
      P2S_CUDA(cudaMemcpyAsync(h->h_t + fo_t, tilt_host + fo_t, 2 * HW * 4, cudaMemcpyHostToDevice, h->s_in));
      P2S_CUDA(cudaEventRecord(h->ev_band, h->s_in));
      P2S_CUDA(cudaStreamWaitEvent(st, h->ev_band, 0));
    }
    s = launch_warp(h, h->d_J, tilt_host ? h->h_t + fo_t : nullptr, h->h_out + fo_img, 1, C, H, W, st);
    if (s != P2S_OK) return s;
    P2S_CUDA(cudaMemcpyAsync(out_host + fo_img, h->h_out + fo_img, (size_t)C * HW * 4, cudaMemcpyDeviceToHost, st));
  }
  P2S_CUDA(cudaStreamSynchronize(st));
  return P2S_OK;
}

p2s_status p2s_debug_profile_buffer(p2s_handle* h, void* device_counters) {
  if (!h) return P2S_ERR_INVALID_ARG;
#if defined(P2S_PROFILE) || defined(P2S_STARTUP_PROF)
  h->prof = (unsigned long long*)device_counters;
  if (h->c1) h->c1->prof = h->prof;
  if (h->seq) h->seq->prof = h->prof;
  return P2S_OK;
#else
  (void)device_counters;
  return P2S_ERR_UNSUPPORTED;
#endif
}

p2s_status p2s_get_info(const p2s_handle* h, p2s_info* info) {
  if (!h || !info) return P2S_ERR_INVALID_ARG;
  info->K = h->K; info->S = h->S; info->n_in = h->n_in; info->h1 = h->h1; info->h2 = h->h2;
  info->n_pad = h->Nk; info->h1_pad = h->N1; info->h2_pad = h->N2; info->in_pad = h->K1;
  info->conv_steps = (int)h->plan.steps.size();
  info->smem_bytes = h->smem_bytes;
  info->kernels_per_render = 2;
  info->stage_bytes = h->stage_bytes;
  info->nring = h->nring;
  info->mlp_backward = h->mb_ok;
  info->c1_plan = h->c1 ? 1 : 0;
  info->c1_smem_bytes = h->c1 ? h->c1->smem_bytes : 0;
  info->c1_nring = h->c1 ? h->c1->nring : 0;
  info->c1_stage_bytes = h->c1 ? h->c1->stage_bytes : 0;
  info->seq_plan = h->seq ? 1 : 0;
  info->seq_nring = h->seq ? h->seq->nring : 0;
  info->seq_stage_bytes = h->seq ? h->seq->stage_bytes : 0;
  return P2S_OK;
}

void p2s_destroy(p2s_handle* h) {
  if (!h) return;
  if (h->c1) p2s_destroy(h->c1);
  if (h->seq) p2s_destroy(h->seq);
  cudaDeviceSynchronize();
  cudaFree(h->d_stream); cudaFree(h->d_items); cudaFree(h->d_mma); cudaFree(h->d_steps); cudaFree(h->d_consts);
  cudaFree(h->d_J);
  cudaFree(h->h_img); cudaFree(h->h_z); cudaFree(h->h_t); cudaFree(h->h_out); cudaFree(h->h_anc);
  cudaFree(h->d_gJ);
  cudaFree(h->d_dib); cudaFree(h->d_ut); cudaFree(h->d_umax);
  cudaFree(h->d_mlpb);
  cudaFree(h->d_col_ws);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->ev_entry) cudaEventDestroy(h->ev_entry);
  if (h->ev_band) cudaEventDestroy(h->ev_band);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  if (h->ev_warped) cudaEventDestroy(h->ev_warped);
  for (cudaEvent_t e : h->ev_rend) cudaEventDestroy(e);
  delete h;
}

}  // extern "C"
