// p2s_adjoint.cuh — dL/dI, the transpose of step a2 ("dI = beta-weighted
// transpose convolution in scatter order"; "differentiable module").
//
// Forward (Eq. 5, reading A2/A4): J_c(p) = sum_k beta_k(p) sum_{i,j} phi_k[i][j]
// I_c[cY(p_y-(i-r))][cX(p_x-(j-r))]. Its transpose, with U_kc = beta_k dL/dJ_c, on the
// clamp-extended grid q in [-r, H+r) x [-r, W+r):
//     dI_pad_c(q) = sum_k sum_{i,j} phi_k[i][j] U_kc(q_y + i - r, q_x + j - r)     (U = 0 outside)
// and dL/dI_c(y, x) = sum of dI_pad_c over the q that clamp to (y, x).
//
// Tensor-core form (one GEMM per band of R output rows, strip of 128 U columns x'):
//     P[x'][(s, j)] = sum_{k, w} U_k(q0 - r + w, x') * phi_k[w - s][j]      (s < R, j < S)
//     dI_pad(q0 + s, x) = sum_j P[x + j - r][(s, j)]                          (the diagonal sum)
// M = 128 columns x' per strip; strips tile U with stride 128 (no halo: each strip adds its partial
// diagonal sums for the 128 + 2r output columns its P rows reach, RED.ADD), contraction (k, window
// row w), WR = ceil8(S + R - 1) window rows per basis function, N = R x S split in two halves of
// Nh columns (two accumulators in TMEM). CTA pairs (cta_group::2, M = 256): each CTA of a pair
// computes its own strip (its 128 rows of the pair UMMA), and the pair shares the B operand --
// each CTA stages half of its N rows -- which halves the dominant traffic (the phi table) per
// CTA. U is row-major fp16 [B*C*K][H][Ws] (written by the
// adjoint fused kernel's epilogue, kAdj = 2); two 3-D TMA boxes (64 columns x window rows x 1
// plane, SWIZZLE_128B) per stage land it as MN-major 128B-swizzled atoms (128 B rows: efficient
// TMA, unlike 16-B core-matrix rows); out-of-range rows/columns read as zeros, so there is no
// halo logic. The B table (phi arranged per (k, w) x (s, j), zero where w - s is outside the
// filter) is one TMA per CTA and stage from an L2-resident table built at p2s_init. The epilogue
// moves one output row's S accumulator columns to shared memory and sums diagonals; results go
// to the clamped pixel with RED.ADD (interior pixels get exactly one add; border pixels collect
// their clamp preimage).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sm100.cuh"
#include "p2s_kernels.cuh"  // u_scale_exp / exp2i (U's range scale)

namespace p2s {

struct alignas(64) DiParams {
  CUtensorMap umap;        // U fp16 [B*C*K][H][Ws] viewed as (x%8, y, x/8, plane)
  CUtensorMap bmap;        // B table as uint8 [rows][256]
  float* gI;               // [B][C][H][W] fp32, zeroed by the caller; RED targets
  const uint32_t* u_maxbits;  // [B*C] U's per-plane range scale (u_scale_exp, p2s_kernels.cuh)
  int BC, K, H, W, S, r;
  int R, nchunk, kg, ngroups, Nh, OW;
  int xs0, nbands, nstrips, npairs, ntiles;  // strip t reads U columns [xs0 + OW t, + 128)
  int a_bytes, b_bytes, stage_bytes, nring, off_p, off_bar;
  int egroups;                                     // epilogue groups (blockDim = 64 + 128 egroups)  // b_bytes: this CTA's half of a stage's B;
                                                            // stage_bytes: a + b rounded up to 1 KB
};

// warp 0 producer, warp 1 MMA (leader) / TMEM, warps 2.. epilogue: kDiGroups groups of four warps
// (one per TMEM lane quadrant), each with its own P buffer, split a tile's output rows (TMEM is
// single-buffered: N = R x S fills it, so the epilogue's row loop is on the tensor pipe's path)
constexpr int kDiGroups = 4;
constexpr int kDiThreads = 64 + 128 * kDiGroups;

// TMA 4-D tile load for a CTA pair: completes on `mbar_cluster` (the leader's barrier)
P2S_DEV void tma2_load_3d(void* dst_smem, const void* tmap, int c0, int c1, int c2, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(mbar_cluster)
      : "memory");
}
// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2 at bits 61-63): for the MN-major U
// tile, LBO = byte offset between the two 64-column (128 B) atoms, SBO = 1024 B between 8-row
// groups; start addresses stay 1 KB aligned.
P2S_DEV uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return sdesc(saddr, lbo_bytes, sbo_bytes) | (2ull << 61);
}

// tile = (plane bc, band, strip pair sp); CTA rank rho takes strip 2 sp + rho
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kDiThreads, 1)
    k_adjoint_image(const __grid_constant__ DiParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int stage_bytes = p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* empty = full + p.nring;
  uint64_t* acc_full = empty + p.nring;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  float* sP = reinterpret_cast<float*>(smem + p.off_p);
  const int warp = (int)warp_id(), lane = (int)lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.nring; ++i) {
      mbar_init(&full[i], 1);   // leader: armed with both CTAs' bytes
      mbar_init(&empty[i], 1);  // both: the leader's commit (multicast)
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 2 * 4 * p.egroups);  // leader: every epilogue warp of both CTAs
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int per_bc = p.nbands * p.npairs;
  const int pair = (int)blockIdx.x >> 1, npair_ctas = (int)gridDim.x >> 1;

  if (warp == 0) {
    // ---------------- producer (both CTAs): this CTA's U chunks + its half of the B slab
    if (lane == 0) {
      prefetch_tmap(&p.umap);
      prefetch_tmap(&p.bmap);
      int s = 0;
      uint32_t ph = 0;
      const int brows = p.b_bytes >> 8;
      for (int t = pair; t < p.ntiles; t += npair_ctas) {
        const int bc = t / per_bc, rem = t - bc * per_bc;
        const int band = rem / p.npairs, sp = rem - band * p.npairs;
        const int q0 = -p.r + band * p.R;                                 // first output row
        const int xb = p.xs0 + (2 * sp + (int)rank) * p.OW;               // first U column
        for (int g = 0; g < p.ngroups; ++g) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * (uint32_t)(p.a_bytes + p.b_bytes));
          const uint32_t mb = cluster_addr(&full[s], 0);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          // the basis function's whole window (nchunk x 8 rows), two 64-column boxes landing as
          // 128B-swizzled MN-major atoms: smem [x/64][row][x%64]
          tma2_load_3d(st, &p.umap, xb, q0 - p.r, bc * p.K + g, mb);
          tma2_load_3d(st + p.a_bytes / 2, &p.umap, xb + 64, q0 - p.r, bc * p.K + g, mb);
          tma2_load_2d(st + p.a_bytes, &p.bmap, 0, (2 * g + (int)rank) * brows, mb);
          if (++s == p.nring) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader, whole warp, elected lane issues the pair UMMAs)
    if (leader) {
      const uint32_t idesc = idesc_f16(256, (uint32_t)p.Nh) | (1u << 15);  // A (U) is MN-major
      const uint32_t smem_base = smem_u32(smem);
      const uint32_t nh2 = (uint32_t)p.Nh / 2u;                          // B rows per CTA
      const uint32_t half_b = (uint32_t)p.nchunk * nh2 * 16u;
      int s = 0;
      uint32_t ph = 0, tl = 0;
      for (int t = pair; t < p.ntiles; t += npair_ctas, ++tl) {
        mbar_wait(acc_empty, (tl & 1) ^ 1);
        tc_fence_after();
        for (int g = 0; g < p.ngroups; ++g) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_base + (uint32_t)(s * stage_bytes);
          const uint32_t b0 = a0 + (uint32_t)p.a_bytes;
          for (int ks = 0; ks < p.nchunk / 2; ++ks) {
            const uint64_t ad = sdesc_sw128(a0 + (uint32_t)ks * 2048u, (uint32_t)p.a_bytes / 2u, 1024u);
            const uint32_t acc = (g > 0 || ks > 0) ? 1u : 0u;
            umma2_f16_elect(tmem, ad, sdesc(b0 + (uint32_t)ks * 2u * nh2 * 16u, nh2 * 16u, 128u), idesc, acc);
            umma2_f16_elect(tmem + (uint32_t)p.Nh, ad,
                            sdesc(b0 + half_b + (uint32_t)ks * 2u * nh2 * 16u, nh2 * 16u, 128u), idesc, acc);
          }
          umma2_commit_elect(&empty[s]);
          if (++s == p.nring) { s = 0; ph ^= 1; }
        }
        umma2_commit_elect(acc_full);
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): TMEM lane m = U column x' = xs + m of this CTA's strip
    const int m = 32 * (warp & 3) + lane;
    const uint32_t tlane = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const int grp = (warp - 2) >> 2;                          // epilogue group
    const int per = (p.R + p.egroups - 1) / p.egroups;         // rows per group (>= 1 each)
    const int sr_begin = min(p.R, grp * per), sr_end = min(p.R, sr_begin + per);
    float* const sPg = sP + (size_t)grp * p.S * 128;
    const int half_r = p.R / 2;
    const size_t HW = (size_t)p.H * p.W;
    uint32_t tl = 0;
    for (int t = pair; t < p.ntiles; t += npair_ctas, ++tl) {
      const int bc = t / per_bc, rem = t - bc * per_bc;
      const int band = rem / p.npairs, sp = rem - band * p.npairs;
      const int strip = 2 * sp + (int)rank;
      const int q0 = -p.r + band * p.R;
      const int x0 = p.xs0 + strip * p.OW;  // this CTA's strip: U / P columns [x0, x0 + 128)
      mbar_wait(acc_full, tl & 1);
      tc_fence_after();
      for (int sr = sr_begin; sr < sr_end; ++sr) {
        const int col = (sr / half_r) * p.Nh + (sr % half_r) * p.S;
        // this output row's S accumulator columns -> sP[j][m], read as 16-aligned column blocks
        for (int jb = col & ~15; jb < col + p.S; jb += 16) {
          float v[16];
          tmem_ld16(tlane + (uint32_t)jb, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int j = jb + i - col;
            if (j >= 0 && j < p.S) sPg[j * 128 + m] = v[i];
          }
        }
        if (sr == sr_end - 1) {  // every accumulator column this group reads: release TMEM
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc_empty, 0);
        }
        named_bar_sync(1 + grp, 128);
        const int qy = q0 + sr;
        if (strip < p.nstrips && qy < p.H + p.r) {
          // the strip's partial diagonal sums for output columns qx = x0 - r + o, o < 128 + 2r:
          // the taps j whose P row x0 + o + j - 2r lies in this strip (the neighbouring strip adds
          // the rest through the same RED), so strips tile U without a halo
          const float un = exp2i(-u_scale_exp(__ldg(p.u_maxbits + bc)));  // undo U's range scale (exact)
          const int y = qy < 0 ? 0 : (qy >= p.H ? p.H - 1 : qy);
          for (int o = m; o < 128 + 2 * p.r; o += 128) {
            const int qx = x0 - p.r + o;
            if (qx < -p.r || qx >= p.W + p.r) continue;
            const int jlo = max(0, 2 * p.r - o), jhi = min(p.S, 128 + 2 * p.r - o);
            const float* row = sPg + (o - 2 * p.r);
            float acc = 0.f;
            for (int j = jlo; j < jhi; ++j) acc += row[j * 129];
            const int x = qx < 0 ? 0 : (qx >= p.W ? p.W - 1 : qx);
            atomicAdd(p.gI + (size_t)bc * HW + (size_t)y * p.W + x, acc * un);
          }
        }
        named_bar_sync(1 + grp, 128);
      }
    }
  }
  // no CTA leaves while its peer's UMMAs may still read its shared memory / TMEM
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc2<512>(tmem);
}

}  // namespace p2s
