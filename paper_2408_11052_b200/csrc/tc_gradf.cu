// tc_gradf.cu — the logits gradient pass (A4) for BOTH sides in one pass over the N x N tile
// grid (BF16 path, W = 1, L2 / dot energy, D = 64).
//
// Paper: InfoNCE fwd/bwd/sym P:619-630 and the logsumexp penalty P:361 / Alg. 1 P:1052 give
// g_ij = dL/dl_ij in closed form (readings A-02..A-05); the energy VJP (App. A.2):
//   L2:  w_ij = g_ij / r_ij,  dPhi_i = sum_j w_ij psi_j - (sum_j w_ij) phi_i
//                             dPsi_j = sum_i w_ij phi_i - (sum_i w_ij) psi_j
//   dot: w_ij = g_ij,         dPhi = W Psi,  dPsi = W^T Phi
// The two-call design (tc_logits.cu) evaluates every w_ij twice, once per orientation.  Here
// one CTA (128 rows x a column split) forms each W tile once and feeds the tcgen05 MMAs:
//   S_t          = A . B_t^T      (M=128 rows, N=128 cols, K=64)
//   dA          += W . B_t        (M=128 rows, N=64, K=128 cols)   TMEM-resident over the split
//   [dB_t | cs_t] = W^T . [A | 1] (M=128 cols, N=80, K=128 rows)   one MMA per K step: the
//                                  all-ones chunk sits 16 KB after A (L2: column sums of w)
// Two epilogue groups of 8 warps ping-pong over the tiles (group t & 1 owns S / W / dB buffer
// t & 1): one group's readout and synchronisation overlap the other's XU work.  S and the
// back-MMAs have separate issuing threads.  dB_t is accumulated across row blocks in a global
// fp32 buffer by TMA bulk-tensor REDUCTIONS (cp.reduce.async.bulk .add.f32 of 16 KB halves
// from swizzled SMEM staging) and cs_t by red.global.add; the row side keeps per-split
// partials; grad_merge2 finishes both sides (the -rs A term, the positive-pair term, fp32 +
// bf16 outputs).  The loss (readings A-02..A-05) is reduced in the same kernel.
// fp32 atomics make the column-side sum order nondeterministic at the 1-ulp level (row side
// and every other stage stay deterministic); the path's tolerance is 2e-2 (north_star).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_gradf.h"
#include "tc_merge.cuh"

namespace crl {
namespace tc {
namespace gf {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsq(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsq_abs(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fabsf(x)));
  return y;
}
// 1/sqrt(|x|) for a PAIR on the FMA pipe: exponent-halving integer guess (one IMAD.HI each),
// two Newton steps y <- y (3/2 - (x/2) y^2) in packed FFMA2 / FMUL2 (relative error ~5e-6)
__device__ __forceinline__ void rsq_pair_fma(float x0, float x1, float& r0, float& r1) {
  x0 = fabsf(x0);
  x1 = fabsf(x1);
  int i0, i1;
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i0) : "r"(__float_as_int(x0)), "r"((int)0x80000000), "r"(0x5f375a86));
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i1) : "r"(__float_as_int(x1)), "r"((int)0x80000000), "r"(0x5f375a86));
  const f32x2 nhx = f2_mul(f2_pack(x0, x1), f2_pack(-0.5f, -0.5f));
  f32x2 y = f2_pack(__int_as_float(i0), __int_as_float(i1));
  const f32x2 c15 = f2_pack(1.5f, 1.5f);
#pragma unroll
  for (int it = 0; it < 2; ++it) y = f2_mul(y, f2_fma(f2_mul(nhx, y), y, c15));
  f2_unpack(y, r0, r1);
}
__device__ __forceinline__ float ex2_neg(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x));
  return y;
}
__device__ __forceinline__ void tmem_ld1_nowait(uint32_t taddr, uint32_t& r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace gf

#ifndef CRL_GF_RSQ_EMU
#define CRL_GF_RSQ_EMU 0
#endif
// of every 4 logit pairs, this many take rsqrt on the FMA pipe instead of the MUFU (measured on
// B200, N = 16384: 0 -> 271 us, 1 -> 270, 2 -> 286, 4 -> 331: not XU-bound, off)
constexpr int kGfRsqEmuPairs = CRL_GF_RSQ_EMU;

struct TcGradFArgs {
  int Na, Nb;
  int cols_per_split;              // multiple of 128
  const float* a_stat;             // [Na]  L2: |a|^2
  const float* b_stat;             // [Nb padded]
  const float* lr;                 // [Na]  row LSE (natural log)
  const float* lc;                 // [Nb padded] column LSE
  const float* lcf;                // [Nb padded] column coefficient (lse_merge / stats_merge)
  const int* fac_ok;
  float c_r, c_c, beta_r, invN;
  float* part_da;                  // [S][Na][64]
  float* part_rs;                  // [S][Na]
  float* cs_acc;                   // [Nb] column sums of w (L2), accumulated
  // the loss (readings A-02..A-05), computed by the otherwise idle warps 2-3 of the column
  // split 0 CTAs (one launch less on the critical path); null loss_part: not here
  const float* phi32; const float* psi32;       // fp32 representations (positives l_ii)
  float* loss_part;                // [row blocks][4] partial sums
  unsigned* loss_ticket;
  float* loss_acc;                 // [3] sums of (LSE_i - l_ii), (LSE'_i - l_ii), LSE_i^2
  float* loss_out;                 // [4] or null
  int *skip, *adam_t, *status;
  float loss_cf, loss_cb, loss_beta;
  int dbg;                         // timing ablations (CRL_GF_DBG): 1 no back-MMAs, 2 no W math, 4 no dB reduce
};

// the loss from the statistics (as optim.cu loss_partial / loss_finalize)
// row block a0 / 128's partial sums -> loss_part; the last row block (ticket) adds them in a
// fixed order and finalises the loss (as optim.cu loss_finalize)
__device__ void gradf_loss_finish(const TcGradFArgs& p, int a0, float s1, float s2, float s3) {
  const int rb = a0 / 128, R = (p.Na + 127) / 128;
  p.loss_part[rb * 4 + 0] = s1;
  p.loss_part[rb * 4 + 1] = s2;
  p.loss_part[rb * 4 + 2] = s3;
  __threadfence();
  if (atomicAdd(p.loss_ticket, 1u) != (unsigned)(R - 1)) return;
  __threadfence();
  float t1 = 0.f, t2 = 0.f, t3 = 0.f;                  // last row block: fixed order, deterministic
  for (int j = 0; j < R; ++j) {
    t1 += __ldcg(p.loss_part + j * 4 + 0); t2 += __ldcg(p.loss_part + j * 4 + 1); t3 += __ldcg(p.loss_part + j * 4 + 2);
  }
  *p.loss_ticket = 0u;
  p.loss_acc[0] = t1; p.loss_acc[1] = t2; p.loss_acc[2] = t3;
  const float Lf = t1 * p.invN, Lb = t2 * p.invN, P = p.loss_beta * t3 * p.invN;
  const bool flat = p.loss_cf < 0.f || p.loss_cb < 0.f;        // FlatNCE: see optim.cu
  const float tot = fabsf(p.loss_cf) * Lf + fabsf(p.loss_cb) * Lb + P;
  if (p.loss_out) {
    p.loss_out[0] = flat ? 0.f : Lf; p.loss_out[1] = flat ? 0.f : Lb; p.loss_out[2] = P;
    p.loss_out[3] = flat ? P : tot;
  }
  const bool bad = !isfinite(tot);
  *p.skip = bad ? 1 : 0;
  if (bad) set_status(p.status, CRL_ENONFINITE);
  else *p.adam_t += 1;
}

// the positive-pair logit l_ii from the fp32 representations (App. A.2)
template <int ENERGY>
__device__ __forceinline__ float gf_diag_logit(float x, float na, float nb) {
  if (ENERGY == CRL_ENERGY_L2) return -sqrtf(x + kEpsL2);
  if (ENERGY == CRL_ENERGY_L2SQ) return -x;
  if (ENERGY == CRL_ENERGY_COS) return x / (fmaxf(sqrtf(na), kEpsCos) * fmaxf(sqrtf(nb), kEpsCos));
  return x;
}

// one warp (warp 3, while the epilogue works through a long column range)
template <int ENERGY>
__device__ void gradf_loss_rows_warp(const TcGradFArgs& p, int a0, int t) {
  float s1 = 0.f, s2 = 0.f, s3 = 0.f;
  for (int r = t; r < 128; r += 32) {
    const int i = a0 + r;
    if (i >= p.Na) break;
    const float4* a = reinterpret_cast<const float4*>(p.phi32 + (size_t)i * 64);
    const float4* b = reinterpret_cast<const float4*>(p.psi32 + (size_t)i * 64);
    float x = 0.f, na = 0.f, nb = 0.f;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      const float4 u = a[k], v = b[k];
      if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) {
        x = fmaf(u.x - v.x, u.x - v.x, x); x = fmaf(u.y - v.y, u.y - v.y, x);
        x = fmaf(u.z - v.z, u.z - v.z, x); x = fmaf(u.w - v.w, u.w - v.w, x);
      } else {
        x = fmaf(u.x, v.x, x); x = fmaf(u.y, v.y, x); x = fmaf(u.z, v.z, x); x = fmaf(u.w, v.w, x);
      }
      if (ENERGY == CRL_ENERGY_COS) {
        na = fmaf(u.x, u.x, na); na = fmaf(u.y, u.y, na); na = fmaf(u.z, u.z, na); na = fmaf(u.w, u.w, na);
        nb = fmaf(v.x, v.x, nb); nb = fmaf(v.y, v.y, nb); nb = fmaf(v.z, v.z, nb); nb = fmaf(v.w, v.w, nb);
      }
    }
    const float l = gf_diag_logit<ENERGY>(x, na, nb);
    const float lr = p.lr[i], lc = p.lc[i];
    s1 += lr - l; s2 += lc - l; s3 += lr * lr;
  }
  s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
  if (t == 0) gradf_loss_finish(p, a0, s1, s2, s3);
}

template <int ENERGY>
__device__ void gradf_loss_rows_epi(const TcGradFArgs& p, int a0, int t) {
  // the 512 epilogue threads, once their tiles are done: 4 threads per row (16 floats each,
  // coalesced 64 B pieces), fixed-order reductions (shuffles, then 16 warp partials)
  __shared__ float red[3][16];
  const int rl = t >> 2, q4 = t & 3;
  const int i = a0 + rl;
  const bool ok = i < p.Na;
  const float4* a = reinterpret_cast<const float4*>(p.phi32 + (size_t)(ok ? i : 0) * 64) + 4 * q4;
  const float4* b = reinterpret_cast<const float4*>(p.psi32 + (size_t)(ok ? i : 0) * 64) + 4 * q4;
  float x = 0.f, na = 0.f, nb = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 u = a[k], v = b[k];
    if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) {
      x = fmaf(u.x - v.x, u.x - v.x, x); x = fmaf(u.y - v.y, u.y - v.y, x);
      x = fmaf(u.z - v.z, u.z - v.z, x); x = fmaf(u.w - v.w, u.w - v.w, x);
    } else {
      x = fmaf(u.x, v.x, x); x = fmaf(u.y, v.y, x); x = fmaf(u.z, v.z, x); x = fmaf(u.w, v.w, x);
    }
    if (ENERGY == CRL_ENERGY_COS) {
      na = fmaf(u.x, u.x, na); na = fmaf(u.y, u.y, na); na = fmaf(u.z, u.z, na); na = fmaf(u.w, u.w, na);
      nb = fmaf(v.x, v.x, nb); nb = fmaf(v.y, v.y, nb); nb = fmaf(v.z, v.z, nb); nb = fmaf(v.w, v.w, nb);
    }
  }
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  if (ENERGY == CRL_ENERGY_COS) {
    na += __shfl_xor_sync(0xffffffffu, na, 1); na += __shfl_xor_sync(0xffffffffu, na, 2);
    nb += __shfl_xor_sync(0xffffffffu, nb, 1); nb += __shfl_xor_sync(0xffffffffu, nb, 2);
  }
  float s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (ok && q4 == 0) {
    const float l = gf_diag_logit<ENERGY>(x, na, nb);
    const float lr = p.lr[i], lc = p.lc[i];
    s1 = lr - l; s2 = lc - l; s3 = lr * lr;
  }
  s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
  if ((t & 31) == 0) { red[0][t >> 5] = s1; red[1][t >> 5] = s2; red[2][t >> 5] = s3; }
  asm volatile("bar.sync 6, 512;" ::: "memory");
  if (t != 0) return;
  s1 = 0.f; s2 = 0.f; s3 = 0.f;
  for (int w = 0; w < 16; ++w) { s1 += red[0][w]; s2 += red[1][w]; s3 += red[2][w]; }
  if (t != 0) return;
  gradf_loss_finish(p, a0, s1, s2, s3);
}


struct GfCfg {
  static constexpr int D = 64, BNT = 128, STAGES = 3;
  static constexpr int NT = 128 + 512;                 // 4 role warps + 2 groups x 2 warpgroups
  static constexpr int NDB = D + 16;                   // dB MMA width: 64 d + 16 ones
  static constexpr uint32_t A_BYTES = 128 * D * 2;       // 16 KB
  static constexpr uint32_t B_BYTES = BNT * D * 2;       // 16 KB
  static constexpr uint32_t W_BYTES = 128 * BNT * 2;     // 32 KB
  static constexpr uint32_t R_BYTES = BNT * D * 4;       // 32 KB fp32 dB staging (2 x 16 KB halves)
  static constexpr uint32_t ONES_BYTES = 128 * 128;      // 16 KB: K=128 rows x 64 bf16 ones
  static constexpr uint32_t STAT_BYTES = BNT * 4;
  static constexpr size_t smem() {
    return 1024 + A_BYTES + ONES_BYTES + STAGES * B_BYTES + 2 * W_BYTES + 2 * R_BYTES + STAGES * 3 * STAT_BYTES +
           3 * 128 * 4 + 256;
  }
};

// Warp roles: 0 TMA producer, 1 S-MMA issuer, 2 back-MMA issuer (+ TMEM owner), 3 the loss
// (split-0 CTAs); 4..19 two epilogue GROUPS of 8 warps that ping-pong over the tiles: group
// g = t & 1 owns S / W / dB buffer g, computes W_t (warpgroup k of the group: tile columns
// [64k, 64k + 64)) and reads dB_{t-2} back out while the other group keeps the XU busy.
template <int ENERGY>
__global__ void __launch_bounds__(GfCfg::NT, 1) tc_gradf_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                const __grid_constant__ CUtensorMap tmB,
                                                                const __grid_constant__ CUtensorMap tmDB,
                                                                TcGradFArgs p) {
  using C = GfCfg;
  constexpr int BNT = C::BNT, STAGES = C::STAGES, D = C::D;
  constexpr bool L2 = ENERGY == CRL_ENERGY_L2;
  constexpr bool SQ = ENERGY == CRL_ENERGY_L2SQ;                 // L2^2: l = -d2, w = 2 g
  constexpr bool DIFF = L2 || SQ;                                // -(sum w) a terms: column sums, row sums
  constexpr bool COS = ENERGY == CRL_ENERGY_COS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // sOnes sits right after sA: the dB MMA reads B = [A | 1] as one MN-major operand whose
  // second 64-wide N chunk (LBO = 16 KB away) is all ones, so its columns 64..79 are the
  // column sums of w (L2) at no extra instruction
  uint8_t* sA = smem;
  uint8_t* sOnes = sA + C::A_BYTES;
  uint8_t* sB = sOnes + C::ONES_BYTES;
  uint8_t* sW = sB + STAGES * C::B_BYTES;
  uint8_t* sR = sW + 2 * C::W_BYTES;
  float* sStat = reinterpret_cast<float*>(sR + 2 * C::R_BYTES);        // [STAGES][3][BNT]
  float* sMerge = sStat + STAGES * 3 * BNT;                            // [3][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMerge + 3 * 128);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* s_full = b_empty + STAGES;   // [2]
  uint64_t* s_empty = s_full + 2;        // [2]
  uint64_t* w_full = s_empty + 2;        // [2]
  uint64_t* w_empty = w_full + 2;        // [2]
  uint64_t* db_full = w_empty + 2;       // [2]
  uint64_t* db_empty = db_full + 2;      // [2]
  uint64_t* da_full = db_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(da_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a0 = blockIdx.x * 128;
  const int split = blockIdx.y;
  const int jbeg = split * p.cols_per_split;
  const int jend = min(p.Nb, jbeg + p.cols_per_split);
  const int ntiles = jend > jbeg ? (jend - jbeg + BNT - 1) / BNT : 0;
  // the row blocks walk their column tiles from staggered starting points: in lockstep they
  // would all TMA-reduce into the same dB tile (and red.add the same column sums) at once
  const int rot = ntiles > 0 ? blockIdx.x % ntiles : 0;
  auto tile_j0 = [&](int t) { const int tt = t + rot; return jbeg + (tt >= ntiles ? tt - ntiles : tt) * BNT; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmDB);
    mbar_init(a_full, 1);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8);
      mbar_init(&w_full[i], 8); mbar_init(&w_empty[i], 1);
      mbar_init(&db_full[i], 1); mbar_init(&db_empty[i], 8);
    }
    mbar_init(da_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  if (DIFF)
    for (int i = threadIdx.x; i < (int)(C::ONES_BYTES / 16); i += blockDim.x)
      reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM columns: S[2] 0..255, dA 256..319, dB[2] (80 wide: d | column sums) 320..479
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_da = tmem + 256;
  pdl_wait();
  pdl_launch();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------------ TMA producer
    mbar_expect_tx(a_full, C::A_BYTES);
    tma_load_2d(sA, &tmA, a_full, 0, a0);
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES;
      mbar_wait(&b_empty[s], ((t / STAGES) & 1) ^ 1);
      const int j0 = tile_j0(t);
      mbar_expect_tx(&b_full[s], C::B_BYTES + 3 * C::STAT_BYTES);
      tma_load_2d(sB + s * C::B_BYTES, &tmB, &b_full[s], 0, j0);
      float* st = sStat + s * 3 * BNT;
      gf::bulk_g2s(st, p.b_stat + j0, C::STAT_BYTES, &b_full[s]);
      gf::bulk_g2s(st + BNT, p.lc + j0, C::STAT_BYTES, &b_full[s]);
      gf::bulk_g2s(st + 2 * BNT, p.lcf + j0, C::STAT_BYTES, &b_full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ S-MMA issuer
    // S_{t+2} is issued as soon as group t & 1 has pulled S_t into registers; the back-MMAs
    // have their own issuing thread, so neither waits behind the other's dependencies
    const uint32_t id_s = idesc_bf16_f32(128, BNT, false, false);
    mbar_wait(a_full, 0);
    const uint32_t a_base = smem_u32(sA);
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES, b = t & 1;
      mbar_wait(&b_full[s], (t / STAGES) & 1);
      mbar_wait(&s_empty[b], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t b_base = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        mma_bf16(tmem + 128 * b, smem_desc_sw128(a_base + ks * 32, 16, 1024),
                 smem_desc_sw128(b_base + ks * 32, 16, 1024), id_s, ks != 0);
      mma_commit(&s_full[b]);
    }
  } else if (warp == 2 && lane == 0) {
    // ------------------------------------------------------------------ back-MMA issuer
    const uint32_t id_da = idesc_bf16_f32(128, D, false, true);      // A = W (K-major), B = B tile (MN)
    const uint32_t id_db = idesc_bf16_f32(128, DIFF ? C::NDB : D, true, true);   // A = W^T, B = [A | 1] (MN)
    mbar_wait(a_full, 0);
    const uint32_t a_base = smem_u32(sA);
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES, b = t & 1;
      mbar_wait(&w_full[b], (t >> 1) & 1);
      mbar_wait(&db_empty[b], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      if (!(p.dbg & 1)) {
        const uint32_t b_base = smem_u32(sB + s * C::B_BYTES);
        const uint32_t w_base = smem_u32(sW + b * C::W_BYTES);
        // dA += W . B_t   (K = the 128 tile columns j: 64-wide chunks of W 16 KB apart)
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const int j = 64 * c + 16 * ks;
            mma_bf16(tm_da, smem_desc_sw128(w_base + c * 16384 + ks * 32, 16, 1024),
                     smem_desc_sw128(b_base + j * 128, BNT * 128, 1024), id_da, (t | c | ks) != 0);
          }
        // [dB_t | cs_t] = W^T . [A | 1]   (K = the 128 tile rows i, 16 per MMA = +2048 B)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16(tmem + 320 + C::NDB * b, smem_desc_sw128(w_base + ks * 2048, 16384, 1024),
                   smem_desc_sw128(a_base + ks * 2048, 16384, 1024), id_db, ks != 0);
      }
      mma_commit(&db_full[b]);
      mma_commit(&w_empty[b]);
      mma_commit(&b_empty[s]);              // S_t finished before W_t could start
    }
    mma_commit(da_full);
  } else if (warp == 3) {
    // short column ranges: the epilogue threads take the loss after their tiles (below)
    if (p.loss_part != nullptr && split == 0 && ntiles > 2) gradf_loss_rows_warp<ENERGY>(p, a0, lane);
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue groups
    const int wgid = (warp - 4) >> 2;                     // 0..3
    const int grp = wgid >> 1;                            // tiles t with t & 1 == grp
    const int k = wgid & 1;                               // 64-column half of the tile
    const int q = warp & 3;                               // TMEM lane quarter
    const int r = q * 32 + lane;                          // row within the tile
    const int row = a0 + r;
    const bool rv = row < p.Na;
    const bool storer = q == 0 && lane == 0;              // issues the reductions of its half
    const uint32_t lq = (uint32_t)(q * 32) << 16;
    const float astat = rv ? p.a_stat[row] : 0.f;
    const float lr2 = rv ? p.lr[row] * gf::kLog2e : INFINITY;      // rows past the batch: p = 0
    const float lr_nat = rv ? p.lr[row] : 0.f;
    const bool fac_fast = *p.fac_ok != 0;
    const float Ei = fac_fast && rv ? gf::ex2(lr2) : 0.f;
    const float Arow = p.invN * p.c_r + 2.f * p.invN * p.beta_r * lr_nat;
    const float cc0 = p.invN * p.c_c;
    const float rmask = rv ? 1.f : 0.f;
    constexpr float L2e2 = gf::kLog2e * gf::kLog2e;
    const float a_l2 = SQ ? astat * gf::kLog2e : (astat + kEpsL2) * L2e2;
    // L2: w = g rs' L.  cos: l = (a.b) r_i s_j and the MMA operand is w' = g r_i s_j (both
    // sides' dot-form partials come out pre-scaled; grad_merge projects them, A-05)
    const float lsc = L2 ? gf::kLog2e : (SQ ? 2.f : (COS ? astat : 1.f));
    const float nLr = -gf::kLog2e * astat;        // cos: -L r_i
    const float EiL = Ei * lsc, ArowL = Arow * lsc, cc0L = cc0 * lsc;
    const uint32_t w_row = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    const uint32_t bar_id = 2 + wgid;
    f32x2 wsum2 = f2_pack(0.f, 0.f);

    // dB_u readout (u & 1 == grp): TMEM -> swizzled SMEM staging (this warpgroup's 32 d
    // columns = one 16 KB half) -> TMA add-reduction into the accumulator
    auto readout = [&](int u) {
      const int bu = u & 1;
      const int j0 = tile_j0(u);
      const uint32_t tdb = tmem + 320 + C::NDB * bu + lq;
      mbar_wait(&db_full[bu], (u >> 1) & 1);
      tc_fence_after();
      uint32_t v[32], cs = 0u;
      tmem_ld32_nowait(tdb + 32 * k, v);           // d columns [32 k, 32 k + 32)
      if (DIFF && k == 0) gf::tmem_ld1_nowait(tdb + D, cs);   // column 64: sum_i w_ij
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&db_empty[bu]);
      if (DIFF && k == 0 && j0 + r < jend) atomicAdd(p.cs_acc + j0 + r, __uint_as_float(cs));
      if (storer) gf::bulk_wait_read0();            // the reduction of u - 2 has read the buffer
      asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      const uint32_t dst = smem_u32(sR + bu * C::R_BYTES + k * 16384) + w_row;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        gf::sts128(dst + (uint32_t)((c ^ (r & 7)) << 4), make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      if (storer && !(p.dbg & 4)) {
        gf::tma_reduce_add_2d(&tmDB, smem_u32(sR + bu * C::R_BYTES + k * 16384), 32 * k, j0);
        gf::bulk_commit();
      }
    };

    for (int t = grp; t < ntiles; t += 2) {
      const int s = t % STAGES, b = t & 1;
      const int j0 = tile_j0(t);
      const int nval = jend - j0;
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      if (t >= 2) mbar_wait(&w_empty[b], ((t >> 1) - 1) & 1);
      const float* bst = sStat + s * 3 * BNT;
      const uint32_t wt = smem_u32(sW + b * C::W_BYTES + k * 16384) + w_row;
      // four instantiations (ragged tile x fast factor path): kernel-uniform choices stay out
      // of the per-logit code.  Fast L2 path, all in log2 units (L = log2 e), pairs of logits
      // per FFMA2 / FMUL2 / FADD2:
      //   d2' = L^2 (|a|^2 + eps + |b|^2 - 2 a.b), rs' = rsqrt(|d2'|) = 1 / (L r)
      //   t   = d2' rs' + lse2_i,  p = 2^-t            (= 2^(l2 - lse2_i))
      //   w   = g / r = p (E_i cc_j + A_i) L rs'       (L folded into E_i, A_i)
      // (|.| and the negation are free MUFU operand modifiers).  Two 32-column sub-chunks;
      // the S buffer is handed back after the second TMEM load.
      auto tile = [&](auto masked, auto fast) {
        constexpr bool MASK = decltype(masked)::value;
        constexpr bool FAST = decltype(fast)::value;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const int c0 = 64 * k + 32 * c;                 // tile column of this sub-chunk
          uint32_t raw[32];
          tmem_ld32_nowait(tmem + 128 * b + lq + c0, raw);
          tmem_ld_wait();
          if (c == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
          }
          float w[32];
          if (p.dbg & 2) {
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = __uint_as_float(raw[i]);
          } else {
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 b4 = gf::lds128f(smem_u32(bst + c0 + 4 * i4));
            const float4 f4 = gf::lds128f(smem_u32(bst + (FAST ? 2 : 1) * BNT + c0 + 4 * i4));
            if (FAST) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int i = 4 * i4 + 2 * h;
                const f32x2 v2 = f2_pack(__uint_as_float(raw[i]), __uint_as_float(raw[i + 1]));
                const f32x2 b2 = h ? f2_pack(b4.z, b4.w) : f2_pack(b4.x, b4.y);
                const f32x2 f2 = h ? f2_pack(f4.z, f4.w) : f2_pack(f4.x, f4.y);
                const f32x2 fac = f2_fma(f2_pack(EiL, EiL), f2, f2_pack(ArowL, ArowL));
                float t0, t1, rs0 = 1.f, rs1 = 1.f;
                if (L2) {
                  const f32x2 d2 = f2_fma(f2_pack(-2.f * L2e2, -2.f * L2e2), v2,
                                          f2_fma(f2_pack(L2e2, L2e2), b2, f2_pack(a_l2, a_l2)));
                  float d0, d1;
                  f2_unpack(d2, d0, d1);
                  if (((2 * i4 + h) & 3) < kGfRsqEmuPairs) {        // rsqrt of this pair on the FMA pipe
                    gf::rsq_pair_fma(d0, d1, rs0, rs1);
                  } else {
                    rs0 = gf::rsq_abs(d0);
                    rs1 = gf::rsq_abs(d1);
                  }
                  f2_unpack(f2_fma(d2, f2_pack(rs0, rs1), f2_pack(lr2, lr2)), t0, t1);
                } else if (SQ) {                          // t = max(d2 L, 0) + lse2_i
                  float d0, d1;
                  f2_unpack(f2_fma(f2_pack(-2.f * gf::kLog2e, -2.f * gf::kLog2e), v2,
                                   f2_fma(f2_pack(gf::kLog2e, gf::kLog2e), b2, f2_pack(a_l2, a_l2))), d0, d1);
                  f2_unpack(f2_add(f2_pack(fmaxf(d0, 0.f), fmaxf(d1, 0.f)), f2_pack(lr2, lr2)), t0, t1);
                } else if (COS) {
                  f2_unpack(f2_fma(f2_mul(v2, b2), f2_pack(nLr, nLr), f2_pack(lr2, lr2)), t0, t1);
                } else {
                  f2_unpack(f2_fma(v2, f2_pack(-gf::kLog2e, -gf::kLog2e), f2_pack(lr2, lr2)), t0, t1);
                }
                if (MASK) {
                  t0 = c0 + i < nval ? t0 : INFINITY;
                  t1 = c0 + i + 1 < nval ? t1 : INFINITY;
                }
                f32x2 wv = f2_mul(f2_pack(gf::ex2_neg(t0), gf::ex2_neg(t1)), fac);
                if (L2) wv = f2_mul(wv, f2_pack(rs0, rs1));
                if (DIFF) wsum2 = f2_add(wsum2, wv);
                if (COS) wv = f2_mul(wv, b2);
                f2_unpack(wv, w[i], w[i + 1]);
              }
            } else {                                      // exact: q = 2^(l2 - lse2'_j)
              const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
              const float ff[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = 4 * i4 + u;
                const float v = __uint_as_float(raw[i]);
                float rs = 1.f, l2v;
                if (L2) {
                  const float d2 = fmaf(-2.f * L2e2, v, fmaf(L2e2, bb[u], a_l2));
                  rs = gf::rsq_abs(d2);
                  l2v = -fabsf(d2) * rs;
                } else if (SQ) {
                  l2v = -fmaxf(fmaf(-2.f * gf::kLog2e, v, fmaf(gf::kLog2e, bb[u], a_l2)), 0.f);
                } else if (COS) {
                  l2v = v * bb[u] * (-nLr);
                } else {
                  l2v = v * gf::kLog2e;
                }
                if (MASK) l2v = c0 + i < nval ? l2v : -INFINITY;
                const float qe = gf::ex2(l2v - ff[u] * gf::kLog2e);
                float wv = fmaf(gf::ex2(l2v - lr2), ArowL, qe * cc0L) * rmask;
                if (L2) wv *= rs;
                if (DIFF) wsum2 = f2_add(wsum2, f2_pack(wv, 0.f));
                if (COS) wv *= bb[u];
                w[i] = wv;
              }
            }
          }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int kk = 32 * c + 8 * u;                 // column within this 64-wide half
            gf::sts128(wt + (uint32_t)((((kk >> 3) ^ (r & 7))) << 4),
                       make_uint4(pack_bf16x2(w[8 * u], w[8 * u + 1]), pack_bf16x2(w[8 * u + 2], w[8 * u + 3]),
                                  pack_bf16x2(w[8 * u + 4], w[8 * u + 5]), pack_bf16x2(w[8 * u + 6], w[8 * u + 7])));
          }
        }
      };
      if (fac_fast) {
        if (nval >= BNT) tile(std::false_type{}, std::true_type{});
        else tile(std::true_type{}, std::true_type{});
      } else {
        if (nval >= BNT) tile(std::false_type{}, std::false_type{});
        else tile(std::true_type{}, std::false_type{});
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_full[b]);
      if (t >= 2) readout(t - 2);
    }
    // the last tile of this group
    const int tl = ntiles - 1 - ((ntiles - 1 - grp) & 1);
    if (tl >= 0) readout(tl);
    // row side: partial row sums of w (L2) and the split's dA
    float ws0, ws1;
    f2_unpack(wsum2, ws0, ws1);
    const float wsum = ws0 + ws1;
    if (wgid > 0) sMerge[(wgid - 1) * 128 + r] = wsum;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (wgid == 0 && rv && DIFF) p.part_rs[(size_t)split * p.Na + row] = wsum + sMerge[r] + sMerge[128 + r] + sMerge[256 + r];
    mbar_wait(da_full, 0);
    tc_fence_after();
    {
      float v[16];
      tmem_ld16(tm_da + lq + 16 * wgid, v);
      if (ntiles == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      if (rv) {
        float* out = p.part_da + ((size_t)split * p.Na + row) * D + 16 * wgid;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(out)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
    if (p.loss_part != nullptr && split == 0 && ntiles <= 2) gradf_loss_rows_epi<ENERGY>(p, a0, threadIdx.x - 128);
    if (storer) gf::bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------------- host side
bool make_map_f32(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);

bool tc_gradf_supports(int D, int energy) {
  return D == 64 && (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_L2SQ || energy == CRL_ENERGY_DOT ||
                     energy == CRL_ENERGY_COS);
}

// column splits minimising the makespan (waves x tiles per CTA) of the rb x S grid, <= 16
int tc_gradf_splits(int Na, int Nb, int num_sms) {
  if (const char* e = std::getenv("CRL_GF_SPLITS")) return std::max(1, std::min(16, std::atoi(e)));
  const int rb = (Na + 127) / 128;
  const int tiles = (Nb + 127) / 128;
  int best = 1;
  long best_cost = -1;
  for (int s = 1; s <= 16 && s <= tiles; ++s) {
    const int cps = (tiles + s - 1) / s;
    const int sp = (tiles + cps - 1) / cps;
    const long waves = ((long)rb * sp + num_sms - 1) / num_sms;
    const long cost = waves * cps;
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = sp; }
  }
  return best;
}

// the column-side accumulator map: db_acc [Nb][64] fp32, TMA-reduced in boxes {32, 128}
bool tc_gradf_map(CUtensorMap* m, float* db_acc, int Nb) { return make_map_f32(m, db_acc, 64, Nb, 64, 32, 128); }

template <int E>
static cudaError_t launch_gf(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& db, const TcGradFArgs& p,
                             int S, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = GfCfg::smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gradf_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.Na + 127) / 128, S);
  return launch_pdl(tc_gradf_kernel<E>, grid, dim3(GfCfg::NT), smem, st, a, b, db, p);
}

cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st);

// Both sides of the gradient.  Row side (A = Phi rows, B = Psi columns): part_da / part_rs
// per split, merged into dA.  Column side: db_acc [Nb][64] and cs_acc [Nb] must be ZERO on
// entry (accumulated by reductions), merged into dB.
cudaError_t tc_grad_fused(int energy, const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mDB, int Na,
                          int Nb, const float* a_stat, const float* b_stat, const float* lse_row, const float* lse_col,
                          const float* fac_col, const int* fac_ok, float c_r, float c_c, float beta_r, float invN,
                          int S, float* part_da, float* part_rs, float* db_acc, float* cs_acc,
                          const __nv_bfloat16* A, const __nv_bfloat16* B, float* dA, __nv_bfloat16* dAb, float* dB,
                          __nv_bfloat16* dBb, const GradfLoss& loss, cudaStream_t st) {
  TcGradFArgs p{};
  p.Na = Na; p.Nb = Nb;
  p.cols_per_split = ((Nb + S - 1) / S + 127) / 128 * 128;
  p.a_stat = a_stat; p.b_stat = b_stat; p.lr = lse_row; p.lc = lse_col; p.lcf = fac_col; p.fac_ok = fac_ok;
  p.c_r = c_r; p.c_c = c_c; p.beta_r = beta_r; p.invN = invN;
  p.part_da = part_da; p.part_rs = part_rs; p.cs_acc = cs_acc;
  p.phi32 = loss.phi32; p.psi32 = loss.psi32; p.loss_part = loss.part; p.loss_ticket = loss.ticket;
  p.loss_acc = loss.acc; p.loss_out = loss.out; p.skip = loss.skip; p.adam_t = loss.adam_t; p.status = loss.status;
  p.loss_cf = loss.c_f; p.loss_cb = loss.c_b; p.loss_beta = loss.beta;
  p.dbg = std::getenv("CRL_GF_DBG") ? std::atoi(std::getenv("CRL_GF_DBG")) : 0;
  cudaError_t e = energy == CRL_ENERGY_L2     ? launch_gf<CRL_ENERGY_L2>(mA, mB, mDB, p, S, st)
                  : energy == CRL_ENERGY_L2SQ ? launch_gf<CRL_ENERGY_L2SQ>(mA, mB, mDB, p, S, st)
                  : energy == CRL_ENERGY_COS  ? launch_gf<CRL_ENERGY_COS>(mA, mB, mDB, p, S, st)
                                             : launch_gf<CRL_ENERGY_DOT>(mA, mB, mDB, p, S, st);
  if (e != cudaSuccess) return e;
  const float Cdiag = invN * (c_r + c_c);
  // row side; column side ("rows" are the B vectors, the pair partner of B_j is A_j): one launch
  const int pre = energy == CRL_ENERGY_COS;        // cos partials carry r_i s_j already
  const GradMergeArgs g0{part_da, part_rs, A, a_stat, B, b_stat, 0, Cdiag, Na, 64, S, dA, dAb, pre};
  const GradMergeArgs g1{db_acc, cs_acc, B, b_stat, A, a_stat, 0, Cdiag, Nb, 64, 1, dB, dBb, pre};
  return launch_grad_merge2(energy, g0, g1, st);
}

}  // namespace tc
}  // namespace crl
