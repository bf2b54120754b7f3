// tc_logits.cu — bf16 tensor-core logits stage (A3 + A4) for the BF16 path.
//
// Paper: energies App. A.2 P:607-617 (L2 = -||phi-psi|| with the sign of P:614, reading A-01;
// dot P:610; cos P:608); InfoNCE fwd/bwd/sym P:619-630; logsumexp penalty P:361, Alg. 1
// P:1052.  Readings A-02..A-06.
//
// Row-owner orientation (A rows, B columns), l_ij = f(A_i, B_j); called with (Phi, Psi) and
// with (Psi, Phi) exactly like the SIMT kernels (logits_simt.cu).  One CTA = 128 rows of A
// x one column split of B.  The N x N logits never leave the SM:
//   S = A . B^T              tcgen05.mma (M=128, N=BNT, K=D), S double-buffered in TMEM
//   epilogue (row per thread, 2 warpgroups split the columns of a tile):
//     LSE : l = f(S), online max / sum of exp2 -> per-split partial (m, s) per row
//     GRAD: g = dL/dl (closed form, A-02..A-05) -> w (energy chain) -> bf16 W tile in SMEM
//   dA += W . B               tcgen05.mma (M=128, N=D, K=BNT): the SMEM B tile that fed S is
//                             re-used as an MN-major operand (same bytes, other descriptor)
// Per-split partials are merged by lse_merge / grad_merge (grad_merge also applies the L2
// "- (sum_j w_ij) A_i" term and the cosine projection, and emits fp32 + bf16 dA).
//
// L2 uses |a|^2 + |b|^2 - 2 a.b on the bf16-rounded vectors (norms of the same rounded
// vectors, clamped at 0): the tolerance of this path is 2e-2 (north_star).
#include "common.cuh"
#include "tc_common.cuh"
#include "tc_merge.cuh"
#include "loss_common.cuh"
#include "tc_gradf.h"

namespace crl {
namespace tc {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct TcLogitsArgs {
  int Na, Nb, row_offset;
  int cols_per_split;              // multiple of BNT
  const float* a_stat;             // [Na]  L2: |a|^2, cos: 1/max(|a|,eps) (bf16-rounded vectors)
  const float* b_stat;             // [Nb padded]  same for B
  const float* lr;                 // GRAD: row statistic (natural log) [Na]
  const float* lc;                 // GRAD: column statistic [Nb padded]
  const float* lcf;                // GRAD: column coefficient 2^(-lc log2 e)(invN c_c + 2 invN beta_c lc)
  const int* fac_ok;               // GRAD: 1 if all row / column factors of the step are normal
  float c_r, c_c, beta_r, beta_c, invN;
  float* part_m;                   // LSE: [S][Na] running max (log2 units)
  float* part_s;                   // LSE: [S][Na] running sum
  float* part_da;                  // GRAD: [S][Na][D]
  float* part_rs;                  // GRAD: [S][Na] row sums of w (L2)
  const int* gate;                 // LSE: if non-null, run only when *gate != 0 (fused-stats fallback)
  // LSE: if ticket is non-null the last of a row block's S split CTAs merges the block's rows
  // itself (no lse_merge launch): lse / fac / fac_ok_out as lse_merge_kernel writes them
  int* ticket;                     // [row blocks], zero between launches (reset by the merger)
  float* lse; float* fac; int* fac_ok_out; float cc0, cc1;
};

template <int D>
struct LgCfg {
  static constexpr int BNT = D <= 128 ? 128 : 64;         // columns per tile
  static constexpr int STAGES = D <= 128 ? 3 : 2;
  static constexpr int KC = D / 64;                       // 64-wide K chunks of A / B
  static constexpr uint32_t A_BYTES = 128 * D * 2;
  static constexpr uint32_t B_BYTES = BNT * D * 2;
  static constexpr uint32_t W_BYTES = 128 * BNT * 2;
  static constexpr uint32_t STAT_BYTES = BNT * 4;
  static constexpr int TMEM_COLS = 512;
  static constexpr size_t smem(bool grad) {
    return 1024 + A_BYTES + STAGES * B_BYTES + (grad ? 2 * W_BYTES : 0) + STAGES * 3 * STAT_BYTES +
           2 * 128 * 4 * 3 + 512;
  }
};

// byte offset of element (row r, k) inside a K-major SW128 tile chunk (rows at 128 B pitch)
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2);
}

// lse[i] = (max_s m + log2(sum_s s * 2^(m_s - max))) * ln 2
__device__ __forceinline__ void lse_merge_row(const float* __restrict__ pm, const float* __restrict__ ps, int Na,
                                              int S, int i, float* __restrict__ lse, float* __restrict__ fac,
                                              int* __restrict__ fac_ok, float cc0, float cc1) {
  float mx = -INFINITY;
  for (int s = 0; s < S; ++s) mx = fmaxf(mx, __ldcg(pm + (size_t)s * Na + i));
  float t = 0.f;
  for (int s = 0; s < S; ++s) {
    const float m = __ldcg(pm + (size_t)s * Na + i);
    if (m != -INFINITY) t += __ldcg(ps + (size_t)s * Na + i) * exp2f(m - mx);
  }
  const float l2 = mx + log2f(t);                        // LSE in log2 units
  lse[i] = l2 * kLn2;
  // column coefficient for the gradient pass in which these rows are the columns:
  // cc = 2^(-LSE log2 e) (cc0 + cc1 LSE); needs 2^(-LSE log2 e) to be a normal float
  const bool ok = l2 > -120.f && l2 < 120.f;
  fac[i] = ok ? exp2f(-l2) * fmaf(cc1, l2 * kLn2, cc0) : 0.f;
  if (!ok) *fac_ok = 0;
}

template <int D, int ENERGY, bool GRAD>
__device__ __forceinline__ void lg_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const TcLogitsArgs& p) {
  using C = LgCfg<D>;
  constexpr int BNT = C::BNT, STAGES = C::STAGES, KC = C::KC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::A_BYTES;
  uint8_t* sW = sB + STAGES * C::B_BYTES;
  float* sStat = reinterpret_cast<float*>(sW + (GRAD ? 2 * C::W_BYTES : 0));   // [STAGES][3][BNT]
  float* sMerge = sStat + STAGES * 3 * BNT;                                     // [3][128] wg-1 partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMerge + 3 * 128);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* s_full = b_empty + STAGES;
  uint64_t* s_empty = s_full + 2;
  uint64_t* w_full = s_empty + 2;
  uint64_t* w_empty = w_full + 2;
  uint64_t* da_full = w_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(da_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a0 = blockIdx.x * 128;
  const int split = blockIdx.y;
  const int jbeg = split * p.cols_per_split;
  const int jend = min(p.Nb, jbeg + p.cols_per_split);
  const int ntiles = jend > jbeg ? (jend - jbeg + BNT - 1) / BNT : 0;
  if (p.gate != nullptr) {          // exact fallback of the fused statistics pass (tc_stats.cu)
    pdl_wait();
    if (*p.gate == 0) { pdl_launch(); return; }
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    mbar_init(a_full, 1);
    // LSE mode: a B stage (and its column statistics) is free once S(t) is computed AND the
    // 8 epilogue warps are done with the statistics; GRAD mode: once dA(t) is computed
    // (which itself waits for the epilogue's W tile).
    for (int s = 0; s < STAGES; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], GRAD ? 1 : 9); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8);
      mbar_init(&w_full[i], 8); mbar_init(&w_empty[i], 1);
    }
    mbar_init(da_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_s[2] = {tmem, tmem + BNT};
  const uint32_t tm_da = tmem + 2 * BNT;
  pdl_wait();
  pdl_launch();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------------ TMA producer
    mbar_expect_tx(a_full, C::A_BYTES);
#pragma unroll
    for (int c = 0; c < KC; ++c) tma_load_2d(sA + c * 128 * 128, &tmA, a_full, 64 * c, a0);
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES;
      mbar_wait(&b_empty[s], ((t / STAGES) & 1) ^ 1);
      const int j0 = jbeg + t * BNT;
      mbar_expect_tx(&b_full[s], C::B_BYTES + (GRAD ? 3 : 1) * C::STAT_BYTES);
      uint8_t* dst = sB + s * C::B_BYTES;
#pragma unroll
      for (int c = 0; c < KC; ++c) tma_load_2d(dst + c * BNT * 128, &tmB, &b_full[s], 64 * c, j0);
      float* st = sStat + s * 3 * BNT;
      bulk_g2s(st, p.b_stat + j0, C::STAT_BYTES, &b_full[s]);
      if (GRAD) {
        bulk_g2s(st + BNT, p.lc + j0, C::STAT_BYTES, &b_full[s]);
        bulk_g2s(st + 2 * BNT, p.lcf + j0, C::STAT_BYTES, &b_full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t id_s = idesc_bf16_f32(128, BNT, false, false);
    const uint32_t id_da = idesc_bf16_f32(128, D, false, true);
    mbar_wait(a_full, 0);
    const uint32_t a_base = smem_u32(sA);
    auto issue_s = [&](int t) {
      const int s = t % STAGES, b = t & 1;
      mbar_wait(&b_full[s], (t / STAGES) & 1);
      mbar_wait(&s_empty[b], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t b_base = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
      for (int c = 0; c < KC; ++c)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_bf16(tm_s[b], smem_desc_sw128(a_base + c * 16384 + ks * 32, 16, 1024),
                   smem_desc_sw128(b_base + c * BNT * 128 + ks * 32, 16, 1024), id_s, (c | ks) != 0);
      mma_commit(&s_full[b]);
      if (!GRAD) mma_commit(&b_empty[s]);
    };
    auto issue_da = [&](int t) {
      const int s = t % STAGES, b = t & 1;
      mbar_wait(&w_full[b], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t b_base = smem_u32(sB + s * C::B_BYTES);
      const uint32_t w_base = smem_u32(sW + b * C::W_BYTES);
#pragma unroll
      for (int c = 0; c < BNT / 64; ++c)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int j = 64 * c + 16 * ks;                  // K index (column of the tile)
          mma_bf16(tm_da, smem_desc_sw128(w_base + c * 16384 + ks * 32, 16, 1024),
                   smem_desc_sw128(b_base + j * 128, BNT * 128, 1024), id_da, (t | c | ks) != 0);
        }
      mma_commit(&w_empty[b]);
      mma_commit(&b_empty[s]);
    };
    for (int t = 0; t < ntiles; ++t) {
      issue_s(t);
      if (GRAD && t > 0) issue_da(t - 1);
    }
    if (GRAD && ntiles > 0) issue_da(ntiles - 1);
    mma_commit(da_full);
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    const int wg = (warp - 4) >> 2;                       // column half of the tile
    const int q = warp & 3;                               // TMEM lane quarter
    const int r = q * 32 + lane;                          // row within the tile
    const int row = a0 + r;
    const bool rv = row < p.Na;
    const float astat = rv ? p.a_stat[row] : 0.f;
    const float lr2 = (GRAD && rv) ? p.lr[row] * kLog2e : 0.f;
    const float lr_nat = (GRAD && rv) ? p.lr[row] : 0.f;
    // q_ij = p_ij * 2^(lr2_i) * 2^(-lc2_j): one MUFU op per logit instead of two, whenever
    // both factors are normal fp32 numbers (else the exact second exp2 is used)
    // fac_ok == 1 <=> every LSE / LSE' of the step gives a normal factor (lse_merge clears it)
    const bool fac_fast = GRAD && *p.fac_ok != 0;
    const float Ei = fac_fast ? ex2(lr2) : 0.f;
    const float Arow = p.invN * p.c_r + 2.f * p.invN * p.beta_r * lr_nat;
    const float cc0 = p.invN * p.c_c, cc1 = 2.f * p.invN * p.beta_c;
    float m2 = -INFINITY, ssum = 0.f, wsum = 0.f;
    constexpr int HALF = BNT / 2;                         // columns per warpgroup per tile
    constexpr int NCH = HALF / 32;                        // x32 TMEM loads per tile
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES, b = t & 1;
      const int j0 = jbeg + t * BNT;
      const int nval = jend - j0;                         // valid columns in this tile
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      // the whole half-tile is pulled out of TMEM at once; the buffer is then handed back
      // to the MMA warp before any arithmetic (overlaps S(t+2) with this epilogue)
      uint32_t raw[NCH][32];
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        tmem_ld32_nowait(tm_s[b] + ((uint32_t)(q * 32) << 16) + wg * HALF + 32 * c, raw[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      if (GRAD && t >= 2) mbar_wait(&w_empty[b], ((t >> 1) - 1) & 1);
      const float* bst = sStat + s * 3 * BNT;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int c0 = wg * HALF + 32 * c;                // column within the tile
        float tv[32], rsv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int jl = c0 + i;
          const float v = __uint_as_float(raw[c][i]);
          float l;
          if (ENERGY == CRL_ENERGY_L2) {
            const float d2 = fmaxf(fmaf(-2.f, v, astat + bst[jl]), 0.f) + kEpsL2;
            rsv[i] = rsq(d2);
            l = -d2 * rsv[i];
          } else if (ENERGY == CRL_ENERGY_L2SQ) {           // F3, App. A.2: -|a - b|^2
            l = -fmaxf(fmaf(-2.f, v, astat + bst[jl]), 0.f);
          } else if (ENERGY == CRL_ENERGY_COS) {
            l = v * astat * bst[jl];
          } else {
            l = v;
          }
          tv[i] = (jl < nval) ? l * kLog2e : -INFINITY;
        }
        if (!GRAD) {
          // chunk-wise online logsumexp: one rescale per 32 columns, no per-element branches
          float cm = tv[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) cm = fmaxf(cm, tv[i]);
          if (cm > m2) { ssum *= ex2(m2 - cm); m2 = cm; }
          if (m2 != -INFINITY) {
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += ex2(tv[i] - m2);
            ssum += acc;
          }
        } else {
          float w[32];
          // g_ij without the delta_ij term (added exactly by grad_merge):
          //   g = p (A_i + E_i cc_j),  A_i = invN c_r + 2 invN beta_r LSE_i,
          //   cc_j = 2^-lse2'_j (invN c_c + 2 invN beta_c LSE'_j)  (precomputed by lse_merge)
          // masked columns have p = 2^-inf = 0.  fac_fast is kernel-uniform; the exact path
          // evaluates q = 2^(t - lse2'_j) with a second exp2 (two separate loops, no predication).
          auto grad_w = [&](int i, float g) {
            float wv;
            if (ENERGY == CRL_ENERGY_L2) wv = g * rsv[i];
            else if (ENERGY == CRL_ENERGY_L2SQ) wv = 2.f * g;  // dl/dphi = -2 (phi - psi)
            else if (ENERGY == CRL_ENERGY_COS) wv = g * bst[c0 + i];
            else wv = g;
            w[i] = wv;
            if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) wsum += wv;
          };
          if (fac_fast) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float pe = ex2(tv[i] - lr2);
              grad_w(i, pe * fmaf(Ei, bst[2 * BNT + c0 + i], Arow));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float lc = bst[BNT + c0 + i];
              const float pe = ex2(tv[i] - lr2);
              const float qe = ex2(tv[i] - lc * kLog2e);
              grad_w(i, fmaf(pe, Arow, qe * fmaf(cc1, lc, cc0)));
            }
          }
          // 32 bf16 of row r -> four 16-byte units of the swizzled W tile
          uint8_t* wt = sW + b * C::W_BYTES + (c0 >> 6) * 16384;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 pk;
            pk.x = pack_bf16x2(w[8 * u + 0], w[8 * u + 1]);
            pk.y = pack_bf16x2(w[8 * u + 2], w[8 * u + 3]);
            pk.z = pack_bf16x2(w[8 * u + 4], w[8 * u + 5]);
            pk.w = pack_bf16x2(w[8 * u + 6], w[8 * u + 7]);
            *reinterpret_cast<uint4*>(wt + sw128_off(r, (c0 & 63) + 8 * u)) = pk;
          }
        }
      }
      if (!GRAD) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_empty[s]);
      } else {
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_full[b]);
      }
    }
    // ---- per-row partial results: warpgroup 1 hands its half to warpgroup 0
    if (wg == 1) {
      sMerge[r] = m2; sMerge[128 + r] = ssum; sMerge[256 + r] = wsum;
    }
    named_sync(1, 256);
    if (wg == 0 && rv) {
      if (!GRAD) {
        const float m2b = sMerge[r], sb = sMerge[128 + r];
        const float mx = fmaxf(m2, m2b);
        float st = 0.f;
        if (m2 != -INFINITY) st += ssum * ex2(m2 - mx);
        if (m2b != -INFINITY) st += sb * ex2(m2b - mx);
        p.part_m[(size_t)split * p.Na + row] = mx;
        p.part_s[(size_t)split * p.Na + row] = st;
      } else {
        if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ)
          p.part_rs[(size_t)split * p.Na + row] = wsum + sMerge[256 + r];
      }
    }
    if (GRAD && wg == 0) {
      mbar_wait(da_full, 0);
      tc_fence_after();
      float* out = p.part_da + ((size_t)split * p.Na + row) * D;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 16) {
        float v[16];
        tmem_ld16(tm_da + ((uint32_t)(q * 32) << 16) + c0, v);
        if (ntiles == 0) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (rv) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4*>(out + c0)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
    }
  }
  if (!GRAD && p.ticket != nullptr) __threadfence();   // partials visible before the ticket
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
  if (!GRAD && p.ticket != nullptr) {
    // the last split CTA of this row block merges its 128 rows (threadfence-reduction pattern)
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(p.ticket + blockIdx.x, 1) == (int)gridDim.y - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (threadIdx.x < 128 && a0 + (int)threadIdx.x < p.Na)
        lse_merge_row(p.part_m, p.part_s, p.Na, gridDim.y, a0 + threadIdx.x, p.lse, p.fac, p.fac_ok_out, p.cc0,
                      p.cc1);
      if (threadIdx.x == 0) p.ticket[blockIdx.x] = 0;
    }
  }
}

template <int D, int ENERGY, bool GRAD>
__global__ void __launch_bounds__(384, 1) tc_logits_kernel(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB,
                                                           TcLogitsArgs p) {
  lg_body<D, ENERGY, GRAD>(tmA, tmB, p);
}

// both sides' statistics (row call on A = Phi, column call on A = Psi) in one launch:
// blockIdx.z picks the side (same grid shape: W = 1 or both sides B_l x N)
template <int D, int ENERGY>
__global__ void __launch_bounds__(384, 1) tc_logits_lse2_kernel(const __grid_constant__ CUtensorMap tmA0,
                                                                const __grid_constant__ CUtensorMap tmB0,
                                                                const __grid_constant__ CUtensorMap tmA1,
                                                                const __grid_constant__ CUtensorMap tmB1,
                                                                const TcLogitsArgs p0, const TcLogitsArgs p1) {
  const bool z = blockIdx.z != 0;
  lg_body<D, ENERGY, false>(z ? tmA1 : tmA0, z ? tmB1 : tmB0, z ? p1 : p0);
}

// --------------------------------------------------------------------------- merges / prep
// Row statistics of the bf16-rounded representations: L2 -> |x|^2, cos -> 1/max(|x|, eps),
// dot -> 0.  One warp per row.
__global__ void rowstat_bf16_kernel(const __nv_bfloat16* __restrict__ x, int N, int D, int energy,
                                    float* __restrict__ out, int* __restrict__ fac_ok, int fac_init) {
  pdl_wait();
  pdl_launch();
  // re-armed every step (fac_init = 0 forces the exact path: CRL_FORCE_EXACT_Q, for tests)
  if (fac_ok != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *fac_ok = fac_init;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= N) return;
  float s = 0.f;
  for (int k = lane; k < D; k += 32) {
    const float v = __bfloat162float(x[(size_t)w * D + k]);
    s = fmaf(v, v, s);
  }
  s = warp_sum(s);
  if (lane == 0)
    out[w] = (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_L2SQ) ? s
             : (energy == CRL_ENERGY_COS ? 1.f / fmaxf(sqrtf(s), kEpsCos) : 0.f);
}

__global__ void lse_merge_kernel(const float* __restrict__ pm, const float* __restrict__ ps, int Na, int S,
                                 float* __restrict__ lse, float* __restrict__ fac, int* __restrict__ fac_ok,
                                 float cc0, float cc1, const int* __restrict__ gate) {
  pdl_wait();
  pdl_launch();
  if (gate != nullptr && *gate == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Na) return;
  lse_merge_row(pm, ps, Na, S, i, lse, fac, fac_ok, cc0, cc1);
}

// dA[i] = sum_s part[s][i]  (+ energy finalisation), fp32 and bf16 outputs.  One warp per row.
// Also adds the positive-pair (delta_ii) term of dL/dl, -C delta_ij with C = invN (c_r + c_c),
// which the tile epilogue leaves out: its energy chain uses the pair (A_i, B_{row_offset+i})
// (L2: 1/r_ii from the difference form; cos: 1/|B_i|).
template <int ENERGY>
__global__ void grad_merge_kernel(const GradMergeArgs g) {
  pdl_wait();
  pdl_launch();
  grad_merge_row<ENERGY>(g, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31);
}
// both sides of the fused gradient pass in one launch: blockIdx.y picks the row / column side;
// the row side's CTAs also reduce the loss when L.part is set (MergeLoss)
template <int ENERGY>
__global__ void grad_merge2_kernel(const GradMergeArgs g0, const GradMergeArgs g1, const MergeLoss L) {
  pdl_wait();
  pdl_launch();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  grad_merge_row<ENERGY>(blockIdx.y ? g1 : g0, w, lane);
  if (blockIdx.y != 0 || L.part == nullptr) return;
  __shared__ float red[3][8];
  __shared__ bool last;
  float s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (w < g0.Na) {
    float l;
    if (g0.D == 256) l = merge_diag_logit<ENERGY, 8>(g0, w, lane);
    else if (g0.D == 128) l = merge_diag_logit<ENERGY, 4>(g0, w, lane);
    else l = merge_diag_logit<ENERGY, 2>(g0, w, lane);
    const float lr = L.lr[w], lc = L.lc[w];
    s1 = lr - l; s2 = lc - l; s3 = lr * lr;
  }
  const int wi = threadIdx.x >> 5;
  if (lane == 0) { red[0][wi] = s1; red[1][wi] = s2; red[2][wi] = s3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t1 = 0.f, t2 = 0.f, t3 = 0.f;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) { t1 += red[0][j]; t2 += red[1][j]; t3 += red[2][j]; }
    L.part[blockIdx.x * 4 + 0] = t1; L.part[blockIdx.x * 4 + 1] = t2; L.part[blockIdx.x * 4 + 2] = t3;
    __threadfence();
    last = atomicAdd(L.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // last row-side CTA: the CTA partials in a fixed order (strided, then a tree): deterministic
  __threadfence();
  __shared__ float tr[3][256];
  float t1 = 0.f, t2 = 0.f, t3 = 0.f;
  for (unsigned j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    t1 += __ldcg(L.part + j * 4 + 0); t2 += __ldcg(L.part + j * 4 + 1); t3 += __ldcg(L.part + j * 4 + 2);
  }
  tr[0][threadIdx.x] = t1; tr[1][threadIdx.x] = t2; tr[2][threadIdx.x] = t3;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h)
      for (int c = 0; c < 3; ++c) tr[c][threadIdx.x] += tr[c][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    L.acc[0] = tr[0][0]; L.acc[1] = tr[1][0]; L.acc[2] = tr[2][0];
    *L.ticket = 0u;                               // re-armed for the next (graph) replay
    if (L.finalize) loss_finalize_dev(L.acc, L.invN, L.c_f, L.c_b, L.beta, L.out, L.skip, L.adam_t, L.status);
  }
}

// ------------------------------------------------------------------------------- host side
bool make_map_bf16(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
cudaError_t launch_grad_merge(int energy, const float* part, const float* prs, const __nv_bfloat16* A,
                              const float* a_stat, const __nv_bfloat16* Bg, const float* b_stat, int row_offset,
                              float Cdiag, int Na, int D, int S, float* out, __nv_bfloat16* outb, cudaStream_t st);

bool tc_logits_supports(int D) { return D == 64 || D == 128 || D == 256; }

int tc_logits_splits(int Na, int Nb, int D, int num_sms) {
  const int rb = (Na + 127) / 128;
  const int bnt = D <= 128 ? 128 : 64;
  const int tiles = (Nb + bnt - 1) / bnt;
  // choose the column split that minimises (waves x tiles per CTA), i.e. the makespan of a
  // static grid of rb x S CTAs on num_sms SMs (<= 8 splits: partial buffers grow with S)
  int best = 1;
  long best_cost = -1;
  for (int s = 1; s <= 8 && s <= tiles; ++s) {
    const int cps = (tiles + s - 1) / s;
    const int sp = (tiles + cps - 1) / cps;
    const long ctas = (long)rb * sp;
    const long waves = (ctas + num_sms - 1) / num_sms;
    const long cost = waves * cps;
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = sp; }
  }
  return best;
}

bool tc_logits_maps(CUtensorMap* mA, CUtensorMap* mB, const __nv_bfloat16* A, int Na, const __nv_bfloat16* B,
                    int Nb, int D) {
  const int bnt = D <= 128 ? 128 : 64;
  return make_map_bf16(mA, A, D, Na, D, 64, 128) && make_map_bf16(mB, B, D, Nb, D, 64, bnt);
}

template <int D, int ENERGY, bool GRAD>
static cudaError_t launch_lg(const CUtensorMap& a, const CUtensorMap& b, const TcLogitsArgs& p, int S,
                             cudaStream_t st) {
  static bool attr = false;
  const size_t smem = LgCfg<D>::smem(GRAD);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_logits_kernel<D, ENERGY, GRAD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.Na + 127) / 128, S);
  return launch_pdl(tc_logits_kernel<D, ENERGY, GRAD>, grid, dim3(384), smem, st, a, b, p);
}

template <bool GRAD>
static cudaError_t dispatch_lg(int D, int energy, const CUtensorMap& a, const CUtensorMap& b,
                               const TcLogitsArgs& p, int S, cudaStream_t st) {
#define CRL_LG(DD)                                                                     \
  if (D == DD) {                                                                       \
    if (energy == CRL_ENERGY_L2) return launch_lg<DD, CRL_ENERGY_L2, GRAD>(a, b, p, S, st); \
    if (energy == CRL_ENERGY_L2SQ) return launch_lg<DD, CRL_ENERGY_L2SQ, GRAD>(a, b, p, S, st); \
    if (energy == CRL_ENERGY_DOT) return launch_lg<DD, CRL_ENERGY_DOT, GRAD>(a, b, p, S, st); \
    return launch_lg<DD, CRL_ENERGY_COS, GRAD>(a, b, p, S, st);                         \
  }
  CRL_LG(64)
  CRL_LG(128)
  CRL_LG(256)
#undef CRL_LG
  return cudaErrorInvalidValue;
}

cudaError_t tc_logits_lse(int D, int energy, const CUtensorMap& mA, const CUtensorMap& mB, int Na, int Nb,
                          const float* a_stat, const float* b_stat, int S, float* part_m, float* part_s,
                          float* lse, float* fac, int* fac_ok, float cc0, float cc1, const int* gate,
                          cudaStream_t st) {
  TcLogitsArgs p{};
  p.Na = Na; p.Nb = Nb;
  const int bnt = D <= 128 ? 128 : 64;
  p.cols_per_split = ((Nb + S - 1) / S + bnt - 1) / bnt * bnt;
  p.a_stat = a_stat; p.b_stat = b_stat; p.part_m = part_m; p.part_s = part_s; p.gate = gate;
  cudaError_t e = dispatch_lg<false>(D, energy, mA, mB, p, S, st);
  if (e != cudaSuccess) return e;
  return launch_pdl(lse_merge_kernel, dim3((Na + 255) / 256), dim3(256), 0, st, (const float*)part_m,
                    (const float*)part_s, Na, S, lse, fac, fac_ok, cc0, cc1, gate);
}

// both sides of the online-max statistics in ONE launch, each row block merged in-kernel by its
// last split CTA (ticket: [2][row blocks] ints, zero on entry and left zero).  c0 / c1: the
// row call (A = Phi) and the column call (A = Psi); same Na, Nb.
cudaError_t tc_logits_lse_pair(int D, int energy, const LseSide& c0, const LseSide& c1, int Na, int Nb, int S,
                               int* fac_ok, int* ticket, const int* gate, cudaStream_t st) {
  TcLogitsArgs p[2]{};
  const int bnt = D <= 128 ? 128 : 64;
  const int rb = (Na + 127) / 128;
  for (int z = 0; z < 2; ++z) {
    const LseSide& c = z ? c1 : c0;
    p[z].Na = Na; p[z].Nb = Nb;
    p[z].cols_per_split = ((Nb + S - 1) / S + bnt - 1) / bnt * bnt;
    p[z].a_stat = c.a_stat; p[z].b_stat = c.b_stat; p[z].part_m = c.part_m; p[z].part_s = c.part_s;
    p[z].gate = gate; p[z].ticket = ticket + z * rb;
    p[z].lse = c.lse; p[z].fac = c.fac; p[z].fac_ok_out = fac_ok; p[z].cc0 = c.cc0; p[z].cc1 = c.cc1;
  }
  auto go = [&](auto kern, size_t smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(rb, S, 2), dim3(384), smem, st, *c0.mA, *c0.mB, *c1.mA, *c1.mB, p[0], p[1]);
  };
#define CRL_LG2(DD)                                                                                   \
  if (D == DD) {                                                                                      \
    const size_t sm = LgCfg<DD>::smem(false);                                                          \
    if (energy == CRL_ENERGY_L2) return go(tc_logits_lse2_kernel<DD, CRL_ENERGY_L2>, sm);              \
    if (energy == CRL_ENERGY_L2SQ) return go(tc_logits_lse2_kernel<DD, CRL_ENERGY_L2SQ>, sm);          \
    if (energy == CRL_ENERGY_DOT) return go(tc_logits_lse2_kernel<DD, CRL_ENERGY_DOT>, sm);            \
    return go(tc_logits_lse2_kernel<DD, CRL_ENERGY_COS>, sm);                                          \
  }
  CRL_LG2(64)
  CRL_LG2(128)
  CRL_LG2(256)
#undef CRL_LG2
  return cudaErrorInvalidValue;
}

cudaError_t tc_logits_grad(int D, int energy, const CUtensorMap& mA, const CUtensorMap& mB, int Na, int Nb,
                           int row_offset, const float* a_stat, const float* b_stat, const float* lr,
                           const float* lc, const float* lcf, float c_r, float c_c, float beta_r, float beta_c,
                           float invN, int S, float* part_da, float* part_rs, const __nv_bfloat16* A,
                           const __nv_bfloat16* Bg, float* dA,
                           __nv_bfloat16* dAb, const int* fac_ok, cudaStream_t st) {
  TcLogitsArgs p{};
  p.Na = Na; p.Nb = Nb; p.row_offset = row_offset;
  const int bnt = D <= 128 ? 128 : 64;
  p.cols_per_split = ((Nb + S - 1) / S + bnt - 1) / bnt * bnt;
  p.a_stat = a_stat; p.b_stat = b_stat; p.lr = lr; p.lc = lc; p.lcf = lcf; p.fac_ok = fac_ok;
  p.c_r = c_r; p.c_c = c_c; p.beta_r = beta_r; p.beta_c = beta_c; p.invN = invN;
  p.part_da = part_da; p.part_rs = part_rs;
  cudaError_t e = dispatch_lg<true>(D, energy, mA, mB, p, S, st);
  if (e != cudaSuccess) return e;
  const float Cdiag = invN * (c_r + c_c);
  return launch_grad_merge(energy, part_da, part_rs, A, a_stat, Bg, b_stat, row_offset, Cdiag, Na, D, S, dA, dAb,
                           st);
}

cudaError_t launch_grad_merge(int energy, const float* part, const float* prs, const __nv_bfloat16* A,
                              const float* a_stat, const __nv_bfloat16* Bg, const float* b_stat, int row_offset,
                              float Cdiag, int Na, int D, int S, float* out, __nv_bfloat16* outb, cudaStream_t st) {
  const GradMergeArgs g{part, prs, A, a_stat, Bg, b_stat, row_offset, Cdiag, Na, D, S, out, outb, 0};
  const dim3 grid((Na * 32 + 255) / 256);
  if (energy == CRL_ENERGY_L2) return launch_pdl(grad_merge_kernel<CRL_ENERGY_L2>, grid, dim3(256), 0, st, g);
  if (energy == CRL_ENERGY_L2SQ) return launch_pdl(grad_merge_kernel<CRL_ENERGY_L2SQ>, grid, dim3(256), 0, st, g);
  if (energy == CRL_ENERGY_COS) return launch_pdl(grad_merge_kernel<CRL_ENERGY_COS>, grid, dim3(256), 0, st, g);
  return launch_pdl(grad_merge_kernel<CRL_ENERGY_DOT>, grid, dim3(256), 0, st, g);
}
// row side (g0) and column side (g1) of the fused gradient pass, one launch (+ the loss when
// loss != nullptr: grad2 path)
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st,
                               const MergeLoss* loss, int nsides) {
  // nsides = 1: g0 only (the caller runs the other side as its own launch, e.g. on another stream)
  const dim3 grid(((nsides == 1 ? g0.Na : max(g0.Na, g1.Na)) * 32 + 255) / 256, nsides == 1 ? 1 : 2);
  const MergeLoss L = loss ? *loss : MergeLoss{};
  if (energy == CRL_ENERGY_L2) return launch_pdl(grad_merge2_kernel<CRL_ENERGY_L2>, grid, dim3(256), 0, st, g0, g1, L);
  if (energy == CRL_ENERGY_L2SQ)
    return launch_pdl(grad_merge2_kernel<CRL_ENERGY_L2SQ>, grid, dim3(256), 0, st, g0, g1, L);
  if (energy == CRL_ENERGY_COS) return launch_pdl(grad_merge2_kernel<CRL_ENERGY_COS>, grid, dim3(256), 0, st, g0, g1, L);
  return launch_pdl(grad_merge2_kernel<CRL_ENERGY_DOT>, grid, dim3(256), 0, st, g0, g1, L);
}
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st,
                               const MergeLoss* loss) {
  return launch_grad_merge2(energy, g0, g1, st, loss, 2);
}
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st) {
  return launch_grad_merge2(energy, g0, g1, st, nullptr, 2);
}

cudaError_t launch_rowstat_bf16(const __nv_bfloat16* x, int N, int D, int energy, float* out, int* fac_ok,
                                int fac_init, cudaStream_t st) {
  return launch_pdl(rowstat_bf16_kernel, dim3((N * 32 + 255) / 256), dim3(256), 0, st, x, N, D, energy, out,
                    fac_ok, fac_init);
}

}  // namespace tc
}  // namespace crl
