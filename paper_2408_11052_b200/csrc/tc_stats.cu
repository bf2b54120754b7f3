// tc_stats.cu — fused row + column logsumexp statistics of the logits (A3) in ONE pass over
// the N x N tile grid, for the bounded energies (L2, cosine) on the BF16 path.
//
// Paper: energies App. A.2 P:607-617 (L2 = -||phi - psi||, reading A-01; cos P:608); the
// InfoNCE forward/backward terms need LSE_i = log sum_j e^{l_ij} (rows) and LSE'_j =
// log sum_i e^{l_ij} (columns) (readings A-02..A-05).
//
// Why one pass suffices: both energies are bounded above by a constant known in advance
// (L2: l <= 0; cos: l <= 1), so e_ij = exp(l_ij) needs no running max: it cannot overflow,
// and ONE exponential per logit feeds both the row sum and the column sum (the two-call
// online-max design of tc_logits.cu evaluates every exponential twice).  Underflow is the
// only hazard (a whole row or column below e^-69, i.e. every distance > 69); stats_merge
// detects it and raises a device flag that runs the exact online-max path instead
// (reading A-29), so the result never silently loses precision.
//
// One CTA = 128 rows of A (Phi) x one column split of B (Psi).  Per 128-column tile:
//   S = A . B^T                    tcgen05.mma (M=128, N=128, K=D) into TMEM (double-buffered)
//   epilogue (thread = row):       e_ij = 2^(l_ij log2 e), row sum in registers, and the bf16
//                                  tile E written to SMEM (SW128, the layout an MN-major
//                                  operand expects)
//   C = 1 . E                      tcgen05.mma (M=128, N=128, K=128 rows) with an all-ones A:
//                                  every row of C holds the 128 column sums of the tile
//   readout (warp 3)               one TMEM row -> colpart[row block][j]
// E is rounded to bf16 for the column-sum MMA (fp32 accumulation): relative error <= 2^-9
// per term, unbiased (round-to-nearest), within the path's 2e-2 tolerance (north_star).
// Row sums stay fp32.  Ragged tiles mask columns j >= N explicitly; rows past the batch are
// masked through their statistic (L2: |a|^2 = 1e30 -> e = 0; cos: additive -inf mask).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"

namespace crl {
namespace tc {
namespace fs {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kMaskBig = 1e30f;

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
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

}  // namespace fs

struct TcStatsArgs {
  int Na, Nb;
  int cols_per_split;              // multiple of 128
  const float* a_stat;             // [Na]  L2: |a|^2, cos: 1/max(|a|, eps)
  const float* b_stat;             // [Nb + pad]
  float* part_rs;                  // [S][Na] row sums of e_ij over this split's columns
  float* colpart;                  // [R][ldc] column sums of e_ij over this CTA's 128 rows
  int ldc;
};

template <int D>
struct StCfg {
  static constexpr int BNT = 128;
  static constexpr int STAGES = D <= 64 ? 3 : 2;
  static constexpr int KC = D / 64;
  static constexpr uint32_t A_BYTES = 128 * D * 2;
  static constexpr uint32_t B_BYTES = BNT * D * 2;
  static constexpr uint32_t E_BYTES = 128 * BNT * 2;     // one bf16 E tile
  static constexpr uint32_t ONES_BYTES = 128 * 128 * 2;  // all-ones A operand (M=128, K=128)
  static constexpr uint32_t STAT_BYTES = BNT * 4;
  static constexpr size_t smem() {
    return 1024 + A_BYTES + STAGES * B_BYTES + 2 * E_BYTES + ONES_BYTES + STAGES * STAT_BYTES + 512 + 256;
  }
};

template <int D, int ENERGY>
__global__ void __launch_bounds__(384, 1) tc_stats_kernel(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB,
                                                          TcStatsArgs p) {
  using C = StCfg<D>;
  constexpr int BNT = C::BNT, STAGES = C::STAGES, KC = C::KC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::A_BYTES;
  uint8_t* sE = sB + STAGES * C::B_BYTES;
  uint8_t* sOnes = sE + 2 * C::E_BYTES;
  float* sStat = reinterpret_cast<float*>(sOnes + C::ONES_BYTES);     // [STAGES][BNT]
  float* sM = sStat + STAGES * BNT;                                   // [128] row-sum hand-off
  uint64_t* bars = reinterpret_cast<uint64_t*>(sM + 128);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* s_full = b_empty + STAGES;    // [2]
  uint64_t* s_empty = s_full + 2;         // [2]
  uint64_t* e_full = s_empty + 2;         // [2]
  uint64_t* e_empty = e_full + 2;         // [2]
  uint64_t* c_full = e_empty + 2;         // [2]
  uint64_t* c_empty = c_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(c_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x;
  const int a0 = rb * 128;
  const int split = blockIdx.y;
  const int jbeg = split * p.cols_per_split;
  const int jend = min(p.Nb, jbeg + p.cols_per_split);
  const int ntiles = jend > jbeg ? (jend - jbeg + BNT - 1) / BNT : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    mbar_init(a_full, 1);
    // a B stage is free once S(t) is computed (MMA commit) and the 8 epilogue warps are done
    // with its column statistics
    for (int s = 0; s < STAGES; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 9); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8);
      mbar_init(&e_full[i], 8); mbar_init(&e_empty[i], 1);
      mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  // all-ones operand (bf16 1.0 = 0x3F80): every layout of it is the same matrix
  for (int i = threadIdx.x; i < (int)(C::ONES_BYTES / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_s[2] = {tmem, tmem + 128};
  const uint32_t tm_c[2] = {tmem + 256, tmem + 384};
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
      mbar_expect_tx(&b_full[s], C::B_BYTES + C::STAT_BYTES);
      uint8_t* dst = sB + s * C::B_BYTES;
#pragma unroll
      for (int c = 0; c < KC; ++c) tma_load_2d(dst + c * BNT * 128, &tmB, &b_full[s], 64 * c, j0);
      fs::bulk_g2s(sStat + s * BNT, p.b_stat + j0, C::STAT_BYTES, &b_full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t id_s = idesc_bf16_f32(128, BNT, false, false);
    const uint32_t id_c = idesc_bf16_f32(128, BNT, false, true);     // B = E is MN-major
    mbar_wait(a_full, 0);
    const uint32_t a_base = smem_u32(sA);
    const uint32_t ones = smem_u32(sOnes);
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
      mma_commit(&b_empty[s]);
    };
    auto issue_c = [&](int t) {
      const int b = t & 1;
      mbar_wait(&e_full[b], (t >> 1) & 1);
      mbar_wait(&c_empty[b], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t e_base = smem_u32(sE + b * C::E_BYTES);
      // K = the 128 rows of E, 16 per MMA (+2048 B in the MN-major SW128 layout); the two
      // 64-column halves of E are 16 KB apart (LBO)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_bf16(tm_c[b], smem_desc_sw128(ones + ks * 32, 16, 1024), smem_desc_sw128(e_base + ks * 2048, 16384, 1024),
                 id_c, ks != 0);
      mma_commit(&c_full[b]);
      mma_commit(&e_empty[b]);
    };
    for (int t = 0; t < ntiles; ++t) {
      issue_s(t);
      if (t > 0) issue_c(t - 1);
    }
    if (ntiles > 0) issue_c(ntiles - 1);
  } else if (warp == 3) {
    // ------------------------------------------------------------------ column-sum readout
    // every TMEM row of C holds the same 128 column sums; this warp reads its lane quarter
    float* out = p.colpart + (size_t)rb * p.ldc;
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1;
      const int j0 = jbeg + t * BNT;
      mbar_wait(&c_full[b], (t >> 1) & 1);
      tc_fence_after();
      uint32_t v[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nowait(tm_c[b] + (96u << 16) + 32 * c, v[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c_empty[b]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t mine = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) mine = (i == lane) ? v[c][i] : mine;
        const int j = j0 + 32 * c + lane;
        if (j < jend) out[j] = __uint_as_float(mine);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    const int wg = (warp - 4) >> 2;                       // 64-column half of the tile
    const int q = warp & 3;                               // TMEM lane quarter
    const int r = q * 32 + lane;                          // row within the tile
    const int row = a0 + r;
    const bool rv = row < p.Na;
    constexpr float L2e2 = fs::kLog2e * fs::kLog2e;
    // L2: d2' = (|a|^2 + |b|^2 - 2 a.b) (log2 e)^2, l2 = -sqrt(d2') (log2 units); rows past
    // the batch get |a|^2 = 1e30 so e = 0.  cos: l2 = a.b (1/|a|)(1/|b|) log2 e + mask_i.
    const float astat = rv ? p.a_stat[row] : fs::kMaskBig;
    const float a_l2 = astat * L2e2;
    const float a_cos = rv ? astat * fs::kLog2e : 0.f;
    const float m_cos = rv ? 0.f : -fs::kMaskBig;
    const uint32_t e_row = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    float rsum = 0.f;
    for (int t = 0; t < ntiles; ++t) {
      const int s = t % STAGES, b = t & 1;
      const int j0 = jbeg + t * BNT;
      const int nval = jend - j0;
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      uint32_t raw[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c)
        tmem_ld32_nowait(tm_s[b] + ((uint32_t)(q * 32) << 16) + wg * 64 + 32 * c, raw[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      if (t >= 2) mbar_wait(&e_empty[b], ((t >> 1) - 1) & 1);
      const uint32_t st_a = smem_u32(sStat + s * BNT + wg * 64);
      const uint32_t e_a = smem_u32(sE + b * C::E_BYTES + wg * 16384) + e_row;
      // two instantiations: full tiles carry no per-element column mask (a uniform `if` inside
      // one loop gets if-converted into a select per element)
      auto tile = [&](auto masked) {
      constexpr bool MASK = decltype(masked)::value;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float e[32];
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) {
          const float4 bs = fs::lds128f(st_a + (uint32_t)(32 * c + 4 * i4) * 4u);
          const float bb[4] = {bs.x, bs.y, bs.z, bs.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = 4 * i4 + u;
            const float v = __uint_as_float(raw[c][i]);
            float l2;
            if (ENERGY == CRL_ENERGY_L2) {
              const float d2 = fmaxf(fmaf(-2.f * L2e2, v, fmaf(L2e2, bb[u], a_l2)), kEpsL2 * L2e2);
              l2 = -d2 * fs::rsq(d2);
            } else {
              l2 = fmaf(v * bb[u], a_cos, m_cos);
            }
            e[i] = fs::ex2(l2);
          }
        }
        if (MASK) {                                       // ragged tile: columns j >= N are not logits
#pragma unroll
          for (int i = 0; i < 32; ++i) e[i] = (wg * 64 + 32 * c + i < nval) ? e[i] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) rsum += e[i];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = 32 * c + 8 * u;                    // column within this 64-wide half
          fs::sts128(e_a + (uint32_t)((((k >> 3) ^ (r & 7))) << 4),
                     make_uint4(pack_bf16x2(e[8 * u], e[8 * u + 1]), pack_bf16x2(e[8 * u + 2], e[8 * u + 3]),
                                pack_bf16x2(e[8 * u + 4], e[8 * u + 5]), pack_bf16x2(e[8 * u + 6], e[8 * u + 7])));
        }
      }
      };
      if (nval >= BNT) tile(std::false_type{});
      else tile(std::true_type{});
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) { mbar_arrive(&e_full[b]); mbar_arrive(&b_empty[s]); }
    }
    // row sums: warpgroup 1 hands its half to warpgroup 0
    if (wg == 1) sM[r] = rsum;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (wg == 0 && rv) p.part_rs[(size_t)split * p.Na + row] = rsum + sM[r];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// LSE from plain sums (the fused pass has no running max: shift 0):
//   threads [0, Na):       LSE_i  = ln sum_s part_rs[s][i]             -> lse_row, fac_row
//   threads [Na, Na + Nb): LSE'_j = ln sum_r colpart[r][j] (or colsum) -> lse_col, fac_col
// fac = 2^-LSE2 (cc0 + cc1 LSE) as in lse_merge (tc_logits.cu).  A sum that is not a normal,
// finite float well above the underflow range sets *bad (exact online-max path runs).
__global__ void stats_merge_kernel(const float* __restrict__ part_rs, int S, int Na, const float* __restrict__ colpart,
                                   int R, int ldc, int Nb, float* __restrict__ lse_row, float* __restrict__ fac_row,
                                   float* __restrict__ lse_col, float* __restrict__ fac_col, int* __restrict__ fac_ok,
                                   int* __restrict__ bad, float rc0, float rc1, float cc0, float cc1,
                                   int force_bad) {
  pdl_wait();
  pdl_launch();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (force_bad && i == 0) atomicExch(bad, 1);         // CRL_FORCE_STATS_FALLBACK (tests)
  float t = 0.f, c0, c1;
  float *lse, *fac;
  if (i < Na) {
    for (int s = 0; s < S; ++s) t += part_rs[(size_t)s * Na + i];
    lse = lse_row; fac = fac_row; c0 = rc0; c1 = rc1;
  } else {
    i -= Na;
    if (i >= Nb) return;
    for (int s = 0; s < R; ++s) t += colpart[(size_t)s * ldc + i];
    lse = lse_col; fac = fac_col; c0 = cc0; c1 = cc1;
  }
  if (!(t >= 0x1p-100f) || !isfinite(t)) atomicExch(bad, 1);
  const float l2 = log2f(t);
  lse[i] = l2 * fs::kLn2;
  const bool ok = l2 > -120.f && l2 < 120.f;
  fac[i] = ok ? exp2f(-l2) * fmaf(c1, l2 * fs::kLn2, c0) : 0.f;
  if (!ok) *fac_ok = 0;
}

// ------------------------------------------------------------------------------- host side
bool tc_stats_supports(int D, int energy) {
  return (D == 64 || D == 128) && (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_COS);
}

int tc_stats_splits(int Na, int Nb, int num_sms) {
  const int rb = (Na + 127) / 128;
  const int tiles = (Nb + 127) / 128;
  int best = 1;
  long best_cost = -1;
  for (int s = 1; s <= 16 && s <= tiles; ++s) {
    const int cps = (tiles + s - 1) / s;
    const int sp = (tiles + cps - 1) / cps;
    const long ctas = (long)rb * sp;
    const long waves = (ctas + num_sms - 1) / num_sms;
    const long cost = waves * cps;
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = sp; }
  }
  return best;
}

template <int D, int ENERGY>
static cudaError_t launch_st(const CUtensorMap& a, const CUtensorMap& b, const TcStatsArgs& p, int S, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = StCfg<D>::smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_stats_kernel<D, ENERGY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.Na + 127) / 128, S);
  return launch_pdl(tc_stats_kernel<D, ENERGY>, grid, dim3(384), smem, st, a, b, p);
}

// One fused statistics pass + merge.  mA/mB: the logits operand maps (A box {64,128},
// B box {64,128}: tc_logits_maps with D <= 128).  part_rs [S][Na], colpart [R][Nb + pad].
cudaError_t tc_stats_fused(int D, int energy, const CUtensorMap& mA, const CUtensorMap& mB, int Na, int Nb,
                           const float* a_stat, const float* b_stat, int S, float* part_rs, float* colpart, int ldc,
                           float* lse_row, float* fac_row, float* lse_col, float* fac_col, int* fac_ok, int* bad,
                           float rc0, float rc1, float cc0, float cc1, cudaStream_t st) {
  TcStatsArgs p{};
  p.Na = Na; p.Nb = Nb;
  p.cols_per_split = ((Nb + S - 1) / S + 127) / 128 * 128;
  p.a_stat = a_stat; p.b_stat = b_stat; p.part_rs = part_rs; p.colpart = colpart; p.ldc = ldc;
  cudaError_t e;
  if (D == 64) e = energy == CRL_ENERGY_L2 ? launch_st<64, CRL_ENERGY_L2>(mA, mB, p, S, st)
                                           : launch_st<64, CRL_ENERGY_COS>(mA, mB, p, S, st);
  else if (D == 128) e = energy == CRL_ENERGY_L2 ? launch_st<128, CRL_ENERGY_L2>(mA, mB, p, S, st)
                                                 : launch_st<128, CRL_ENERGY_COS>(mA, mB, p, S, st);
  else return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  const int R = (Na + 127) / 128;
  return launch_pdl(stats_merge_kernel, dim3((Na + Nb + 255) / 256), dim3(256), 0, st, (const float*)part_rs, S, Na,
                    (const float*)colpart, R, ldc, Nb, lse_row, fac_row, lse_col, fac_col, fac_ok, bad, rc0, rc1,
                    cc0, cc1, std::getenv("CRL_FORCE_STATS_FALLBACK") ? 1 : 0);
}

}  // namespace tc
}  // namespace crl
