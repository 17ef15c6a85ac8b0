// p2s_host.cu — the C ABI of include/p2s.h: validation, asset packing, execution plan and
// launches of the sm_100a kernels in p2s_kernels.cuh. No torch types, no oracle code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "p2s.h"
#include "p2s_kernels.cuh"

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
  int npos_y = 0, npos_x = 0, chan_bytes = 0;
};

ConvPlan plan_conv(int S) {
  ConvPlan P;
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
  P.npos_y = nblk ? 128 + S + 1 : 0;
  P.npos_x = nex ? 128 + 16 * Pairs : 0;
  const uint32_t ystride = (uint32_t)P.npos_y * 16, xbase = (uint32_t)nblk * ystride;
  P.chan_bytes = (int)(xbase + (uint32_t)nex * P.npos_x * 16);
  for (int g = 0; g < ngroups; ++g)
    for (int b = 0; b < S; ++b) {
      ConvStep st{(uint32_t)(2 * g) * ystride + (uint32_t)b * 16, ystride, {}};
      for (int kk = 0; kk < 16; ++kk) {
        const int a = 16 * g + 8 * (kk / 8) + (kk % 8);
        st.tap[kk] = a < S ? Tap{a, b} : Tap{-1, -1};
      }
      P.steps.push_back(st);
    }
  if (left == 2) {
    const int a0 = 16 * nv16;
    for (int b = 0; b < S; b += 2) {
      ConvStep st{(uint32_t)(nblk - 1) * ystride + (uint32_t)b * 16, 16, {}};
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
      ConvStep st{xbase + (uint32_t)e * P.npos_x * 16 + (uint32_t)b0 * 16, 128, {}};
      for (int kk = 0; kk < 16; ++kk)
        st.tap[kk] = (b0 + kk < S) ? Tap{P.ex_a[e], b0 + kk} : Tap{-1, -1};
      P.steps.push_back(st);
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
  std::vector<StageDesc> stages;
  int nst_l[4];
  int stage_bytes, nring, smem_bytes;
  int off_ring, off_a1, off_a2, off_e, off_tab, off_bar, a1_sbo, a2_sbo;
  int sm_count;
  uint8_t* d_stream = nullptr;
  StageDesc* d_stages = nullptr;
  uint2* d_steps = nullptr;
  float *d_b1 = nullptr, *d_b2 = nullptr, *d_b3 = nullptr, *d_s = nullptr;
  float* d_J = nullptr;
  size_t J_cap = 0;
  float *h_img = nullptr, *h_z = nullptr, *h_t = nullptr, *h_out = nullptr;  // device staging (host path)
  size_t stage_px_cap = 0, stage_chw_cap = 0;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
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

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b) return false;
  const char *pa = (const char*)a, *pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

FusedParams make_params(const p2s_handle* h, int B, int C, int H, int W, int mode) {
  FusedParams p{};
  p.B = B; p.C = C; p.H = H; p.W = W; p.n_in = h->n_in;
  p.nstrips = (W + kTileM - 1) / kTileM;
  p.ntiles = B * p.nstrips * H;
  p.mode = mode;
  p.stream = h->d_stream;
  p.stages = h->d_stages;
  for (int i = 0; i < 4; ++i) p.nst_l[i] = h->nst_l[i];
  p.nstages = h->nst_l[0] + h->nst_l[1] + h->nst_l[2] + h->nst_l[3];
  p.conv_steps = h->d_steps;
  p.nconv = (int)h->plan.steps.size();
  p.b1 = h->d_b1; p.b2 = h->d_b2; p.b3 = h->d_b3; p.svec = h->d_s;
  p.K = h->K; p.Nk = h->Nk; p.K1 = h->K1; p.N1 = h->N1; p.N2 = h->N2; p.r = h->r;
  p.n_ey = (int)h->plan.ey_a0.size(); p.n_ex = (int)h->plan.ex_a.size();
  p.npos_y = h->plan.npos_y; p.npos_x = h->plan.npos_x;
  for (int i = 0; i < p.n_ey; ++i) p.ey_a0[i] = h->plan.ey_a0[i];
  for (int i = 0; i < p.n_ex; ++i) p.ex_a[i] = h->plan.ex_a[i];
  p.chan_bytes = h->plan.chan_bytes;
  p.stage_bytes = h->stage_bytes; p.nring = h->nring;
  p.off_ring = h->off_ring; p.off_a1 = h->off_a1; p.off_a2 = h->off_a2; p.off_e = h->off_e;
  p.off_tab = h->off_tab; p.off_bar = h->off_bar; p.smem_bytes = h->smem_bytes;
  p.a1_sbo = h->a1_sbo; p.a2_sbo = h->a2_sbo;
  return p;
}

p2s_status launch_fused(p2s_handle* h, const FusedParams& p, cudaStream_t st) {
  if (p.ntiles == 0) return P2S_OK;
  const int grid = std::min(h->sm_count, p.ntiles);
  k_fused_p2s<<<grid, kThreads, h->smem_bytes, st>>>(p);
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

p2s_status p2s_init(const p2s_basis* basis, const p2s_mlp* mlp, p2s_handle** out_handle) {
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
  h->K = K; h->S = S; h->r = (S - 1) / 2;
  h->n_in = mlp->n_in; h->h1 = mlp->h1; h->h2 = mlp->h2;
  h->Nk = up16(K); h->K1 = up16(mlp->n_in); h->N1 = up16(mlp->h1); h->N2 = up16(mlp->h2);
  h->plan = plan_conv(S);
  h->sm_count = prop.multiProcessorCount;
  const ConvPlan& P = h->plan;

  // ---- shared-memory layout (E sized for C = 3)
  const int nconv = (int)P.steps.size();
  const int a1_bytes = kTileM * h->K1 * 2;
  const int kh = std::max(h->N1, h->N2);
  const int a2_bytes = kTileM * kh * 2;
  const int e_bytes = 3 * P.chan_bytes;
  const int tab_bytes = kMaxStages * (int)sizeof(StageDesc) + nconv * 8;
  const int bar_bytes = (8 + 2 * 4) * 8 + 16;
  const int fixed = a1_bytes + a2_bytes + e_bytes + tab_bytes + bar_bytes + 4 * 128;
  const int ring_avail = kSmemLimit - fixed;
  int nring = 4, sb = 0;
  for (nring = 4; nring >= 2; --nring) {
    sb = std::min(32768, (ring_avail / nring) / 1024 * 1024);
    if (sb >= 16384 || nring == 2) break;
  }
  const int max_slab = std::max(std::max(h->N1, h->N2), h->Nk) * 32;
  if (sb < max_slab || nconv > kMaxConvSteps) { delete h; return P2S_ERR_UNSUPPORTED; }
  h->nring = nring;
  h->stage_bytes = sb;
  int off = 0;
  h->off_ring = off; off += nring * sb;
  h->off_a1 = off; off += (a1_bytes + 127) / 128 * 128;
  h->off_a2 = off; off += (a2_bytes + 127) / 128 * 128;
  h->off_e = off; off += (e_bytes + 127) / 128 * 128;
  h->off_tab = off; off += (tab_bytes + 127) / 128 * 128;
  h->off_bar = off; off += (8 + 2 * nring) * 8 + 16;
  h->smem_bytes = off;
  h->a1_sbo = (h->K1 / 8) * 128;
  h->a2_sbo = (kh / 8) * 128;
  if (h->smem_bytes > kSmemLimit) { delete h; return P2S_ERR_UNSUPPORTED; }

  // ---- pack the streamed B operands: [W1 slabs][W2 slabs][W3 slabs][conv slabs]
  const int n_slabs[4] = {h->K1 / 16, h->N1 / 16, h->N2 / 16, nconv};
  const int rows[4] = {h->N1, h->N2, h->Nk, h->Nk};
  size_t layer_off[4], total = 0;
  for (int l = 0; l < 4; ++l) { layer_off[l] = total; total += (size_t)n_slabs[l] * rows[l] * 32; }
  std::vector<__half> stream(total / 2, __float2half(0.f));
  auto put = [&](int l, int ks, int n, int kk, float v) {
    stream[layer_off[l] / 2 + (size_t)ks * rows[l] * 16 + slab_idx(n, kk)] = __float2half_rn(v);
  };
  for (int ks = 0; ks < n_slabs[0]; ++ks)
    for (int n = 0; n < h->h1; ++n)
      for (int kk = 0; kk < 16; ++kk) {
        const int k = ks * 16 + kk;
        if (k < h->n_in) put(0, ks, n, kk, mlp->W1[(size_t)n * h->n_in + k]);
      }
  for (int ks = 0; ks < n_slabs[1]; ++ks)
    for (int n = 0; n < h->h2; ++n)
      for (int kk = 0; kk < 16; ++kk) {
        const int k = ks * 16 + kk;
        if (k < h->h1) put(1, ks, n, kk, mlp->W2[(size_t)n * h->h1 + k]);
      }
  for (int ks = 0; ks < n_slabs[2]; ++ks)
    for (int n = 0; n < K; ++n)
      for (int kk = 0; kk < 16; ++kk) {
        const int k = ks * 16 + kk;
        if (k < h->h2) put(2, ks, n, kk, mlp->W3[(size_t)n * h->h2 + k]);
      }
  for (int g = 0; g < nconv; ++g)
    for (int n = 0; n < K; ++n)
      for (int kk = 0; kk < 16; ++kk) {
        const Tap t = P.steps[g].tap[kk];
        if (t.a < 0) continue;
        // psi[a][b] = phi[S-1-a][S-1-b]  (true convolution, A2)
        put(3, g, n, kk, basis->taps[((size_t)n * S + (S - 1 - t.a)) * S + (S - 1 - t.b)]);
      }
  // ---- stage list
  for (int l = 0; l < 4; ++l) {
    const int slab = rows[l] * 32;
    const int per = std::max(1, sb / slab);
    h->nst_l[l] = 0;
    for (int s0 = 0; s0 < n_slabs[l]; s0 += per) {
      const int ns = std::min(per, n_slabs[l] - s0);
      h->stages.push_back(StageDesc{(uint32_t)(layer_off[l] + (size_t)s0 * slab), (uint32_t)(ns * slab),
                                    (uint32_t)l, (uint32_t)s0});
      h->nst_l[l]++;
    }
  }
  if ((int)h->stages.size() > kMaxStages) { delete h; return P2S_ERR_UNSUPPORTED; }
  // ---- biases (zero-padded), tap sums s_k = sum phi_k (for the centred-image identity)
  std::vector<float> b1(h->N1, 0.f), b2(h->N2, 0.f), b3(h->Nk, 0.f), sv(h->Nk, 0.f);
  for (int i = 0; i < h->h1; ++i) b1[i] = mlp->b1[i];
  for (int i = 0; i < h->h2; ++i) b2[i] = mlp->b2[i];
  for (int i = 0; i < K; ++i) {
    b3[i] = mlp->b3[i];
    double s = 0.0;
    for (int t = 0; t < S * S; ++t) s += basis->taps[(size_t)i * S * S + t];
    sv[i] = (float)s;
  }
  std::vector<uint2> steps(nconv);
  for (int g = 0; g < nconv; ++g) steps[g] = make_uint2(P.steps[g].off, P.steps[g].lbo);

  auto fail = [&](p2s_status s) { p2s_destroy(h); return s; };
  cudaError_t e;
#define UP(dst, src, bytes)                                                        \
  if ((e = cudaMalloc(&(dst), (bytes))) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc")); \
  if ((e = cudaMemcpy((dst), (src), (bytes), cudaMemcpyHostToDevice)) != cudaSuccess) \
    return fail(cuda_fail(e, "cudaMemcpy"));
  UP(h->d_stream, stream.data(), total);
  UP(h->d_stages, h->stages.data(), h->stages.size() * sizeof(StageDesc));
  UP(h->d_steps, steps.data(), steps.size() * sizeof(uint2));
  UP(h->d_b1, b1.data(), b1.size() * 4);
  UP(h->d_b2, b2.data(), b2.size() * 4);
  UP(h->d_b3, b3.data(), b3.size() * 4);
  UP(h->d_s, sv.data(), sv.size() * 4);
#undef UP
  if ((e = cudaFuncSetAttribute(k_fused_p2s, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) !=
      cudaSuccess)
    return fail(cuda_fail(e, "cudaFuncSetAttribute"));
  *out_handle = h;
  return P2S_OK;
}

p2s_status p2s_reserve(p2s_handle* h, int B, int C, int H, int W) {
  if (!h || B < 1 || C < 1 || H < 1 || W < 1) return P2S_ERR_INVALID_ARG;
  return ensure_J(h, (size_t)B * C * H * W);
}

p2s_status p2s_set_profile_events(p2s_handle* h, p2s_event_t ev_begin, p2s_event_t ev_end) {
  if (!h || ((ev_begin == nullptr) != (ev_end == nullptr))) return P2S_ERR_INVALID_ARG;
  h->ev_begin = (cudaEvent_t)ev_begin;
  h->ev_end = (cudaEvent_t)ev_end;
  return P2S_OK;
}

static p2s_status render_impl(p2s_handle* h, p2s_image im, const float* z, const float* tilt, float* out,
                              float* J_out, cudaStream_t st) {
  const size_t n_img = (size_t)im.B * im.C * im.H * im.W;
  const size_t n_z = (size_t)im.B * h->n_in * im.H * im.W;
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
  p.zernike = z;
  p.J = J;
  if (h->ev_begin) P2S_CUDA(cudaEventRecord(h->ev_begin, st));
  p2s_status s = launch_fused(h, p, st);
  if (s != P2S_OK) return s;
  if (h->ev_end) P2S_CUDA(cudaEventRecord(h->ev_end, st));
  if (out) {
    const size_t npx = (size_t)im.B * im.H * im.W;
    const int grid = (int)std::min<size_t>((npx + 255) / 256, (size_t)h->sm_count * 16);
    k_tilt_warp<<<grid, 256, 0, st>>>(J, tilt, out, im.B, im.C, im.H, im.W);
    P2S_CUDA(cudaPeekAtLastError());
  }
  return P2S_OK;
}

p2s_status p2s_render(p2s_handle* h, p2s_image im, const float* zernike_field, const float* tilt_field,
                      float* out, p2s_stream_t stream) {
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  if (!zernike_field || !out) return P2S_ERR_INVALID_ARG;
  return render_impl(h, im, zernike_field, tilt_field, out, nullptr, (cudaStream_t)stream);
}

p2s_status p2s_debug_blur(p2s_handle* h, p2s_image im, const float* zernike_field, float* J_out,
                          p2s_stream_t stream) {
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
  FusedParams p = make_params(h, B, 1, H, W, 1);
  p.zernike = zernike_field;
  p.beta_out = beta_out;
  return launch_fused(h, p, (cudaStream_t)stream);
}

p2s_status p2s_render_host(p2s_handle* h, const float* image_host, int B, int C, int H, int W,
                           const float* zernike_host, const float* tilt_host, float* out_host,
                           p2s_stream_t stream) {
  if (!h || !image_host || !zernike_host || !out_host) return P2S_ERR_INVALID_ARG;
  p2s_image im{nullptr, B, C, H, W};
  im.data = image_host;  // validated below against the device copy
  p2s_status s = check_image(h, im);
  if (s != P2S_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t px = (size_t)B * H * W, chw = px * C;
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
  P2S_CUDA(cudaMemcpyAsync(h->h_img, image_host, chw * 4, cudaMemcpyHostToDevice, st));
  P2S_CUDA(cudaMemcpyAsync(h->h_z, zernike_host, px * h->n_in * 4, cudaMemcpyHostToDevice, st));
  if (tilt_host) P2S_CUDA(cudaMemcpyAsync(h->h_t, tilt_host, px * 2 * 4, cudaMemcpyHostToDevice, st));
  im.data = h->h_img;
  s = render_impl(h, im, h->h_z, tilt_host ? h->h_t : nullptr, h->h_out, nullptr, st);
  if (s != P2S_OK) return s;
  P2S_CUDA(cudaMemcpyAsync(out_host, h->h_out, chw * 4, cudaMemcpyDeviceToHost, st));
  P2S_CUDA(cudaStreamSynchronize(st));
  return P2S_OK;
}

p2s_status p2s_get_info(const p2s_handle* h, p2s_info* info) {
  if (!h || !info) return P2S_ERR_INVALID_ARG;
  info->K = h->K; info->S = h->S; info->n_in = h->n_in; info->h1 = h->h1; info->h2 = h->h2;
  info->n_pad = h->Nk; info->h1_pad = h->N1; info->h2_pad = h->N2; info->in_pad = h->K1;
  info->conv_steps = (int)h->plan.steps.size();
  info->smem_bytes = h->smem_bytes;
  info->kernels_per_render = 2;
  return P2S_OK;
}

void p2s_destroy(p2s_handle* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  cudaFree(h->d_stream); cudaFree(h->d_stages); cudaFree(h->d_steps);
  cudaFree(h->d_b1); cudaFree(h->d_b2); cudaFree(h->d_b3); cudaFree(h->d_s);
  cudaFree(h->d_J);
  cudaFree(h->h_img); cudaFree(h->h_z); cudaFree(h->h_t); cudaFree(h->h_out);
  delete h;
}

}  // extern "C"
