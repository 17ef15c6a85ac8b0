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
// M = 128 columns x' (each strip yields OW = floor8(128 - 2r) outputs), contraction (k, window
// row w), WR = ceil8(S + R - 1) window rows per basis function, N = R x S split in two halves of
// Nh columns (two accumulators in TMEM). CTA pairs (cta_group::2, M = 256): each CTA of a pair
// computes its own strip (its 128 rows of the pair UMMA), and the pair shares the B operand --
// each CTA stages half of its N rows -- which halves the dominant traffic (the phi table) per
// CTA. U is row-major fp16 [B*C*K][H][Ws] (written by the
// adjoint fused kernel's epilogue, kAdj = 2); a 4-D TMA view (x%8, y, x/8, plane) with box
// (8, 8, 16, 1) lands one 8-row chunk as MN-major core matrices (8 columns = 16 B by 8 rows),
// M-blocks 128 B apart (SBO), chunks 2 KB apart (LBO); out-of-range rows/columns read as zeros,
// so there is no halo logic, and strips start at multiples of 8 columns (the x%8 coordinate is
// always 0). The B table (phi arranged per (k, w) x (s, j), zero where w - s is outside the
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
  int a_bytes, b_bytes, nring, off_p, off_bar;  // b_bytes: this CTA's half of a stage's B
};

constexpr int kDiThreads = 192;  // warp 0 producer, warp 1 MMA (leader) / TMEM, warps 2-5 epilogue

// TMA 4-D tile load for a CTA pair: completes on `mbar_cluster` (the leader's barrier)
P2S_DEV void tma2_load_4d(void* dst_smem, const void* tmap, int c0, int c1, int c2, int c3, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar_cluster)
      : "memory");
}

// tile = (plane bc, band, strip pair sp); CTA rank rho takes strip 2 sp + rho
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kDiThreads, 1)
    k_adjoint_image(const __grid_constant__ DiParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int stage_bytes = p.a_bytes + p.b_bytes;
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
    mbar_init(acc_empty, 8);  // leader: every epilogue warp of both CTAs
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
        const int xb = (p.xs0 + (2 * sp + (int)rank) * p.OW) >> 3;        // first U column / 8
        for (int g = 0; g < p.ngroups; ++g) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * (uint32_t)stage_bytes);
          const uint32_t mb = cluster_addr(&full[s], 0);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          // the basis function's whole window (nchunk x 8 rows) in one box: smem [x/8][row][x%8]
          tma2_load_4d(st, &p.umap, 0, q0 - p.r, xb, bc * p.K + g, mb);
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
            const uint64_t ad = sdesc(a0 + (uint32_t)ks * 256u, 128u, (uint32_t)p.nchunk * 128u);
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
    const int half_r = p.R / 2;
    const size_t HW = (size_t)p.H * p.W;
    uint32_t tl = 0;
    for (int t = pair; t < p.ntiles; t += npair_ctas, ++tl) {
      const int bc = t / per_bc, rem = t - bc * per_bc;
      const int band = rem / p.npairs, sp = rem - band * p.npairs;
      const int strip = 2 * sp + (int)rank;
      const int q0 = -p.r + band * p.R;
      const int qx = p.xs0 + strip * p.OW + p.r + m;  // this thread's output column
      mbar_wait(acc_full, tl & 1);
      tc_fence_after();
      for (int sr = 0; sr < p.R; ++sr) {
        const int col = (sr / half_r) * p.Nh + (sr % half_r) * p.S;
        // this output row's S accumulator columns -> sP[j][m], read as 16-aligned column blocks
        for (int jb = col & ~15; jb < col + p.S; jb += 16) {
          float v[16];
          tmem_ld16(tlane + (uint32_t)jb, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int j = jb + i - col;
            if (j >= 0 && j < p.S) sP[j * 128 + m] = v[i];
          }
        }
        if (sr == p.R - 1) {  // every accumulator column read: release TMEM to the next tile
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc_empty, 0);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int qy = q0 + sr;
        if (m < p.OW && strip < p.nstrips && qy < p.H + p.r && qx >= -p.r && qx < p.W + p.r) {
          float acc = 0.f;
          for (int j = 0; j < p.S; ++j) acc += sP[j * 128 + m + j];
          acc *= exp2i(-u_scale_exp(__ldg(p.u_maxbits + bc)));  // undo U's range scale (exact)
          const int y = qy < 0 ? 0 : (qy >= p.H ? p.H - 1 : qy);
          const int x = qx < 0 ? 0 : (qx >= p.W ? p.W - 1 : qx);
          atomicAdd(p.gI + (size_t)bc * HW + (size_t)y * p.W + x, acc);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
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
