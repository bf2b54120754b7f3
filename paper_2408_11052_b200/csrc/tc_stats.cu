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
// Persistent kernel: one CTA per SM walks work units (row block rb of 128 rows of A = Phi,
// column chunk ch of B = Psi); the TMEM / barrier pipeline runs across unit boundaries (the A
// tile is double-buffered).  Per 128-column tile:
//   S = A . B^T                    tcgen05.mma (M=128, N=128, K=D) into TMEM (double-buffered)
//   epilogue (thread = row, 4 warpgroups x 32 columns): e_ij = 2^(l_ij log2 e) with packed
//                                  FFMA2 / FADD2 math, row sums in registers, the bf16 tile E
//                                  written to SMEM (SW128, the layout an MN-major operand expects)
//   C = 1 . E                      tcgen05.mma (M=128, N=128, K=128 rows) with an all-ones A:
//                                  every row of C holds the 128 column sums of the tile
//   readout (warp 3)               one TMEM row -> colpart[rb][j]
// Row sums of a unit -> part_rs[ch][row]; stats_merge adds the chunks and the row blocks.
// E is rounded to bf16 for the column-sum MMA (fp32 accumulation): relative error <= 2^-9
// per term, unbiased (round-to-nearest), within the path's 2e-2 tolerance (north_star).
// Ragged tiles mask columns j >= N explicitly; rows past the batch are masked through their
// statistic (L2: |a|^2 = 1e30 -> e = 0; cos: additive -1e30 mask).
#include <cstdio>
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
// sqrt(|x|) for a PAIR on the FMA pipe: y ~ 1/sqrt from the exponent-halving integer guess
// (one IMAD.HI each: magic + floor(-bits / 2)), two Newton steps y <- y (3/2 - (x/2 y) y) in
// packed FFMA2 / FMUL2 (relative error ~5e-6; x = 0 gives 0), then sqrt = x y
__device__ __forceinline__ void sqrt_pair_fma(float x0, float x1, float& r0, float& r1) {
  x0 = fabsf(x0);
  x1 = fabsf(x1);
  int i0, i1;
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i0) : "r"(__float_as_int(x0)), "r"((int)0x80000000), "r"(0x5f375a86));
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i1) : "r"(__float_as_int(x1)), "r"((int)0x80000000), "r"(0x5f375a86));
  const f32x2 x = f2_pack(x0, x1);
  const f32x2 nhx = f2_mul(x, f2_pack(-0.5f, -0.5f));
  f32x2 y = f2_pack(__int_as_float(i0), __int_as_float(i1));
  const f32x2 c15 = f2_pack(1.5f, 1.5f);
#pragma unroll
  for (int it = 0; it < 2; ++it) y = f2_mul(y, f2_fma(f2_mul(nhx, y), y, c15));
  f2_unpack(f2_mul(x, y), r0, r1);
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
  int n_chunks;                    // column chunks per row block (work unit = (rb, chunk))
  int tiles_per_chunk;             // 128-column tiles per chunk
  int n_units;                     // row blocks x n_chunks
  const float* a_stat;             // [Na]  L2: |a|^2, cos: 1/max(|a|, eps)
  const float* b_stat;             // [Nb + pad]
  float* part_rs;                  // [n_chunks][Na] row sums of e_ij over one chunk
  float* colpart;                  // [R][ldc] column sums of e_ij over one row block
  int ldc;
  int trace;                       // measurement: clock64 trace of CTA 0 (CRL_STATS_TRACE)
};

constexpr int kStNWG = 4;          // epilogue warpgroups
#ifndef CRL_ST_NS
#define CRL_ST_NS 2
#endif
constexpr int kNS = CRL_ST_NS;     // S accumulators in TMEM (2 or 3: 128 columns each; 3 measured equal at netscale)
#ifndef CRL_ST_EMU
#define CRL_ST_EMU 0
#endif
// of every 4 logit pairs, this many exp2 pairs skip the MUFU (measured on B200 at N = 16384:
// 1 of 4 is neutral, 186 -> 185 us: the tile loop is latency- not XU-throughput-bound)
constexpr int kStEmuPairs = CRL_ST_EMU;
#ifndef CRL_ST_SQRT_EMU
#define CRL_ST_SQRT_EMU 0
#endif
// of every 4 logit pairs, this many take sqrt on the FMA pipe (Newton) instead of the MUFU
// (measured on B200 at N = 16384: 0 -> 194 us, 1 -> 199, 2 -> 200, 4 -> 251: the kernel is
// issue / latency- rather than XU-bound, so moving work to the FMA pipe does not pay)
constexpr int kStSqrtPairs = CRL_ST_SQRT_EMU;

template <int D>
struct StCfg {
  static constexpr int BNT = 128;
  static constexpr int KC = D / 64;                      // 64-wide K chunks of A / B
  // the B tile is staged in PIECES of up to 2 chunks (D = 256: two 32 KB pieces per tile), so
  // the ring holds more tiles' worth of look-ahead than whole 64 KB tiles would
  static constexpr int PC = KC < 2 ? KC : 2;             // chunks per piece
  static constexpr int NP = KC / PC;                     // pieces per tile
  static constexpr int STAGES = D <= 64 ? 3 : (D <= 128 ? 2 : 3);   // pieces in flight
  static constexpr int ABUF = D <= 128 ? 2 : 1;          // row-block A tiles (double-buffered when small)
  static constexpr int NE = D <= 128 ? 2 : 1;            // bf16 E tiles
  static constexpr uint32_t A_BYTES = 128 * D * 2;
  static constexpr uint32_t P_BYTES = BNT * 64 * 2 * PC; // one B piece
  static constexpr uint32_t E_BYTES = 128 * BNT * 2;     // one bf16 E tile
  static constexpr uint32_t ONES_BYTES = 128 * 64 * 2;   // all-ones A operand chunk (re-used for K 64..127)
  static constexpr uint32_t STAT_BYTES = BNT * 4;
  static constexpr size_t smem() {
    return 1024 + ABUF * A_BYTES + STAGES * P_BYTES + NE * E_BYTES + ONES_BYTES + 2 * STAT_BYTES + 3 * 512 + 256;
  }
};

template <int D, int ENERGY>
__global__ void __launch_bounds__(128 + 128 * kStNWG, 1) tc_stats_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                        const __grid_constant__ CUtensorMap tmB,
                                                                        TcStatsArgs p) {
  using C = StCfg<D>;
  constexpr int BNT = C::BNT, STAGES = C::STAGES, KC = C::KC, PC = C::PC, NP = C::NP, ABUF = C::ABUF, NE = C::NE;
  constexpr int NWG = kStNWG, CW = BNT / NWG, NCH = CW / 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                                 // [ABUF] row-block tiles
  uint8_t* sB = sA + ABUF * C::A_BYTES;                               // [STAGES] B pieces
  uint8_t* sE = sB + STAGES * C::P_BYTES;                             // [NE] E tiles
  uint8_t* sOnes = sE + NE * C::E_BYTES;
  float* sStat = reinterpret_cast<float*>(sOnes + C::ONES_BYTES);     // [2][BNT] column statistics
  float* sM = sStat + 2 * BNT;                                        // [NWG-1][128] row-sum hand-off
  uint64_t* bars = reinterpret_cast<uint64_t*>(sM + 3 * 128);
  uint64_t* a_full = bars;                // [2]
  uint64_t* a_empty = a_full + 2;         // [2]
  uint64_t* b_full = a_empty + 2;         // [STAGES]
  uint64_t* b_empty = b_full + STAGES;    // [STAGES]
  uint64_t* s_full = b_empty + STAGES;    // [kNS]
  uint64_t* s_empty = s_full + kNS;       // [kNS]
  uint64_t* e_full = s_empty + kNS;       // [2]
  uint64_t* e_empty = e_full + 2;         // [2]
  uint64_t* c_full = e_empty + 2;         // [2]
  uint64_t* c_empty = c_full + 2;         // [2]
  uint64_t* st_full = c_empty + 2;        // [2]
  uint64_t* st_empty = st_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(st_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  // the units of this CTA: u = blockIdx.x + k G; unit u = (rb, ch), tiles [ch tpc, (ch+1) tpc)
  auto unit_rb = [&](int u) { return u / p.n_chunks; };
  auto unit_j0 = [&](int u) { return (u % p.n_chunks) * p.tiles_per_chunk * BNT; };
  auto unit_ntiles = [&](int u) {
    const int j0 = unit_j0(u);
    const int j1 = min(p.Nb, j0 + p.tiles_per_chunk * BNT);
    return j1 > j0 ? (j1 - j0 + BNT - 1) / BNT : 0;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < 2; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    // a B piece is free once the S MMAs that read it completed; the column statistics of a
    // tile have their own 2-slot ring, freed by the epilogue warps
    for (int s = 0; s < STAGES; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    for (int i = 0; i < kNS; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4 * NWG); }
    for (int i = 0; i < 2; ++i) {

      mbar_init(&e_full[i], 4 * NWG); mbar_init(&e_empty[i], 1);
      mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], 4);
      mbar_init(&st_full[i], 1); mbar_init(&st_empty[i], 4 * NWG);
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
  const uint32_t tm_s[3] = {tmem, tmem + 128, tmem + 384};   // kNS S accumulators (C sits at 256..287)
  const uint32_t tm_c[2] = {tmem + 256, tmem + 272};   // [128 columns j (lanes)] x 16 (column 0 used)
  pdl_wait();
  pdl_launch();
  __shared__ long long s_tr[4][16];
  const bool trace = p.trace && blockIdx.x == 0;
  if (trace && threadIdx.x == 0) s_tr[0][0] = clock64();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------------ TMA producer
    int g = 0, k = 0, pc = 0;
    for (int u = blockIdx.x; u < p.n_units; u += G, ++k) {
      const int ua = k % ABUF;
      mbar_wait(&a_empty[ua], ((k / ABUF) & 1) ^ 1);
      mbar_expect_tx(&a_full[ua], C::A_BYTES);
#pragma unroll
      for (int c = 0; c < KC; ++c) tma_load_2d(sA + ua * C::A_BYTES + c * 16384, &tmA, &a_full[ua], 64 * c, unit_rb(u) * 128);
      const int nt = unit_ntiles(u), j00 = unit_j0(u);
      for (int t = 0; t < nt; ++t, ++g) {
        const int j0 = j00 + t * BNT;
        const int sb = g & 1;
        mbar_wait(&st_empty[sb], ((g >> 1) & 1) ^ 1);
        mbar_expect_tx(&st_full[sb], C::STAT_BYTES);
        fs::bulk_g2s(sStat + sb * BNT, p.b_stat + j0, C::STAT_BYTES, &st_full[sb]);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp, ++pc) {
          const int s = pc % STAGES;
          mbar_wait(&b_empty[s], ((pc / STAGES) & 1) ^ 1);
          mbar_expect_tx(&b_full[s], C::P_BYTES);
          uint8_t* dst = sB + s * C::P_BYTES;
#pragma unroll
          for (int c = 0; c < PC; ++c) tma_load_2d(dst + c * BNT * 128, &tmB, &b_full[s], 64 * (pp * PC + c), j0);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t id_s = idesc_bf16_f32(128, BNT, false, false);
    // column sums as C^T = E^T 1: A = E^T (MN-major: M = the 128 columns j), B = ones (K-major,
    // N = 16): per tile 8 N = 16 MMAs reading 36 KB of SMEM (the 1 E form read 64 KB into a
    // 128-column accumulator whose rows were all equal)
    const uint32_t id_c = idesc_bf16_f32(128, 16, true, false);
    const uint32_t ones = smem_u32(sOnes);
    auto issue_c = [&](int g) {
      const int b = g & 1, eb = g % NE;
      mbar_wait(&e_full[eb], (g / NE) & 1);
      mbar_wait(&c_empty[b], ((g >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t e_base = smem_u32(sE + eb * C::E_BYTES);
      // K = the 128 rows of E, 16 per MMA (+2048 B in the MN-major SW128 layout); the two
      // 64-column halves of E are 16 KB apart (LBO); the ones chunk serves both K halves
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_bf16(tm_c[b], smem_desc_sw128(e_base + ks * 2048, 16384, 1024), smem_desc_sw128(ones + (ks & 3) * 32, 16, 1024),
                 id_c, ks != 0);
      mma_commit(&c_full[b]);
      mma_commit(&e_empty[eb]);
    };
    int g = 0, k = 0, pc = 0;
    for (int u = blockIdx.x; u < p.n_units; u += G, ++k) {
      const int ua = k % ABUF;
      mbar_wait(&a_full[ua], (k / ABUF) & 1);
      const uint32_t a_base = smem_u32(sA + ua * C::A_BYTES);
      const int nt = unit_ntiles(u);
      if (nt == 0) mma_commit(&a_empty[ua]);                // empty chunk: hand the A buffer back
      for (int t = 0; t < nt; ++t, ++g) {
        const int b = g % kNS;
        mbar_wait(&s_empty[b], ((g / kNS) & 1) ^ 1);
        if (trace && g < 15) s_tr[1][g + 1] = clock64();
#pragma unroll
        for (int pp = 0; pp < NP; ++pp, ++pc) {
          const int s = pc % STAGES;
          mbar_wait(&b_full[s], (pc / STAGES) & 1);
          tc_fence_after();
          const uint32_t b_base = smem_u32(sB + s * C::P_BYTES);
#pragma unroll
          for (int c = 0; c < PC; ++c)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              mma_bf16(tm_s[b], smem_desc_sw128(a_base + (pp * PC + c) * 16384 + ks * 32, 16, 1024),
                       smem_desc_sw128(b_base + c * BNT * 128 + ks * 32, 16, 1024), id_s, (pp | c | ks) != 0);
          mma_commit(&b_empty[s]);
        }
        mma_commit(&s_full[b]);
        if (t == nt - 1) mma_commit(&a_empty[ua]);        // last S of the unit read this A tile
        if (g > 0) issue_c(g - 1);
      }
    }
    if (g > 0) issue_c(g - 1);
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    // NWG warpgroups split the 128 columns of a tile (CW each): 4 warps per SMSP hide the
    // MUFU / TMEM latencies of the per-logit chain
    const int wg = (warp - 4) >> 2;                       // column group of the tile
    const int q = warp & 3;                               // TMEM lane quarter
    const int r = q * 32 + lane;                          // row within the tile
    constexpr float L2e2 = fs::kLog2e * fs::kLog2e;
    const uint32_t e_row = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    const int cg0 = wg * CW;                              // first column of this group
    // column sums of tile x (C(x) in TMEM lane j = column j): read by warpgroup x % NWG two
    // tiles later (C(x) is long complete by then), one 32x32b.x1 TMEM load per warp
    int cs_rb[2] = {0, 0}, cs_j0[2] = {0, 0}, cs_jend[2] = {0, 0};   // tile x's unit, by x & 1
    auto read_cs = [&](int x) {
      const int bx = x & 1;
      mbar_wait(&c_full[bx], (x >> 1) & 1);
      tc_fence_after();
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm_c[bx] + ((uint32_t)(q * 32) << 16)));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c_empty[bx]);
      const int j = cs_j0[bx] + q * 32 + lane;
      if (j < cs_jend[bx]) p.colpart[(size_t)cs_rb[bx] * p.ldc + j] = __uint_as_float(v);
    };
    int g = 0;
    for (int u = blockIdx.x; u < p.n_units; u += G) {
      const int row = unit_rb(u) * 128 + r;
      const bool rv = row < p.Na;
      // L2: d2' = (|a|^2 + |b|^2 - 2 a.b) (log2 e)^2, e = 2^-sqrt(d2') (log2 units); rows
      // past the batch get |a|^2 = 1e30 so e = 0.  cos: l2 = a.b (1/|a|)(1/|b|) log2 e + mask
      const float astat = rv ? p.a_stat[row] : fs::kMaskBig;
      // L2^2: x = d2 log2 e is the negated log2-unit logit, e = 2^-max(x, 0)
      constexpr bool DIFF = ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ;
      constexpr float kx = ENERGY == CRL_ENERGY_L2SQ ? fs::kLog2e : L2e2;
      const f32x2 kL2 = f2_pack(kx, kx);
      const f32x2 kM2 = DIFF ? f2_pack(-2.f * kx, -2.f * kx)
                             : f2_pack(rv ? 0.f : -fs::kMaskBig, rv ? 0.f : -fs::kMaskBig);
      const float ka = DIFF ? astat * kx : (rv ? astat * fs::kLog2e : 0.f);
      const f32x2 kA2 = f2_pack(ka, ka);
      f32x2 racc[2] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
      const int nt = unit_ntiles(u), j00 = unit_j0(u);
      const int jend = min(p.Nb, j00 + p.tiles_per_chunk * BNT);
      for (int t = 0; t < nt; ++t, ++g) {
        const int b = g & 1, eb = g % NE;
        const int nval = jend - (j00 + t * BNT);
        if (g >= 2 && wg == (g - 2) % NWG) read_cs(g - 2);
        cs_rb[b] = unit_rb(u); cs_j0[b] = j00 + t * BNT; cs_jend[b] = jend;   // (tile g - 2's slot is read)
        const int sb = g % kNS;
        mbar_wait(&st_full[b], (g >> 1) & 1);
        mbar_wait(&s_full[sb], (g / kNS) & 1);
        if (trace && threadIdx.x == 128 && g < 15) s_tr[2][g + 1] = clock64();
        tc_fence_after();
        uint32_t raw[NCH][32];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tmem_ld32_nowait(tm_s[sb] + ((uint32_t)(q * 32) << 16) + cg0 + 32 * c, raw[c]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        const uint32_t st_a = smem_u32(sStat + b * BNT + cg0);
        const uint32_t e_a = smem_u32(sE + eb * C::E_BYTES + (cg0 >> 6) * 16384) + e_row;
        // two instantiations: full tiles carry no per-element column mask (a uniform `if`
        // inside one loop gets if-converted into a select per element)
        auto tile = [&](auto masked) {
          constexpr bool MASK = decltype(masked)::value;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            float e[32];
            // pairs of logits per FFMA2 / FADD2 (sm_100 packed fp32); L2: e = 2^-sqrt(|d2'|)
            // (|.| and the negation are free MUFU operand modifiers, sqrt(0) = 0 needs no
            // epsilon: the oracle's sqrt(d2 + 1e-12) differs by <= 1e-6)
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
              const float4 bs = fs::lds128f(st_a + (uint32_t)(32 * c + 4 * i4) * 4u);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int i = 4 * i4 + 2 * h;
                const f32x2 v2 = f2_pack(__uint_as_float(raw[c][i]), __uint_as_float(raw[c][i + 1]));
                const f32x2 b2 = h ? f2_pack(bs.z, bs.w) : f2_pack(bs.x, bs.y);
                float x0, x1;
                if (ENERGY == CRL_ENERGY_L2) {
                  f2_unpack(f2_fma(kM2, v2, f2_fma(kL2, b2, kA2)), x0, x1);
                  if (((2 * i4 + h) & 3) < kStSqrtPairs) {      // sqrt of this pair on the FMA pipe
                    float r0, r1;
                    fs::sqrt_pair_fma(x0, x1, r0, r1);
                    e[i] = ex2_neg(r0);
                    e[i + 1] = ex2_neg(r1);
                  } else if (((2 * i4 + h) & 3) < kStEmuPairs) {       // exp2 of this pair on FMA / ALU
                    ex2_pair_fma(-sqrt_abs(x0), -sqrt_abs(x1), e[i], e[i + 1]);
                  } else {
                    e[i] = ex2_neg(sqrt_abs(x0));
                    e[i + 1] = ex2_neg(sqrt_abs(x1));
                  }
                } else if (ENERGY == CRL_ENERGY_L2SQ) {
                  f2_unpack(f2_fma(kM2, v2, f2_fma(kL2, b2, kA2)), x0, x1);
                  e[i] = ex2_neg(fmaxf(x0, 0.f));
                  e[i + 1] = ex2_neg(fmaxf(x1, 0.f));
                } else {
                  f2_unpack(f2_fma(f2_mul(v2, b2), kA2, kM2), x0, x1);
                  e[i] = fs::ex2(x0);
                  e[i + 1] = fs::ex2(x1);
                }
              }
            }
            if (MASK) {                                   // ragged tile: columns j >= N are not logits
#pragma unroll
              for (int i = 0; i < 32; ++i) e[i] = (cg0 + 32 * c + i < nval) ? e[i] : 0.f;
            }
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) racc[k2 & 1] = f2_add(racc[k2 & 1], f2_pack(e[2 * k2], e[2 * k2 + 1]));
            // E(g) overwrites E(g - NE): wait for that tile's column-sum MMA only now, after
            // this chunk's exponentials (waiting first serialised the math behind the MMA)
            if (c == 0 && g >= NE) mbar_wait(&e_empty[eb], ((g / NE) - 1) & 1);
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4) {
              const int kk = (cg0 & 63) + 32 * c + 8 * v4;   // column within the 64-wide chunk
              fs::sts128(e_a + (uint32_t)((((kk >> 3) ^ (r & 7))) << 4),
                         make_uint4(pack_bf16x2(e[8 * v4], e[8 * v4 + 1]), pack_bf16x2(e[8 * v4 + 2], e[8 * v4 + 3]),
                                    pack_bf16x2(e[8 * v4 + 4], e[8 * v4 + 5]),
                                    pack_bf16x2(e[8 * v4 + 6], e[8 * v4 + 7])));
            }
          }
        };
        if (nval >= BNT) tile(std::false_type{});
        else tile(std::true_type{});
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) { mbar_arrive(&e_full[eb]); mbar_arrive(&st_empty[b]); }
        if (trace && threadIdx.x == 128 && g < 15) s_tr[3][g + 1] = clock64();
      }
      // row sums of the unit: warpgroups 1.. hand their partial sums to warpgroup 0
      float r0, r1, r2, r3;
      f2_unpack(racc[0], r0, r1);
      f2_unpack(racc[1], r2, r3);
      const float rsum = (r0 + r1) + (r2 + r3);
      if (wg > 0) sM[(wg - 1) * 128 + r] = rsum;
      asm volatile("bar.sync 1, %0;" ::"n"(128 * NWG) : "memory");
      if (wg == 0 && rv) {
        float tot = rsum;
#pragma unroll
        for (int gg = 1; gg < NWG; ++gg) tot += sM[(gg - 1) * 128 + r];
        p.part_rs[(size_t)(u % p.n_chunks) * p.Na + row] = tot;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(128 * NWG) : "memory");   // sM reusable
    }
    for (int x = g - 2 < 0 ? 0 : g - 2; x < g; ++x)
      if (wg == x % NWG) read_cs(x);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (trace && threadIdx.x == 0)
    for (int k = 1; k < 4; ++k)
      for (int t = 1; t < 16; ++t) printf("STATS_TRACE %d %d %lld\n", k, t - 1, s_tr[k][t] - s_tr[0][0]);
}

// LSE from plain sums (the fused pass has no running max: shift 0):
//   threads [0, Na):       LSE_i  = ln sum_s part_rs[s][i]   -> lse_row, fac_row
//   threads [Na, Na + Nb): LSE'_j = ln sum_r colpart[r][j]   -> lse_col, fac_col
// fac = 2^-LSE2 (cc0 + cc1 LSE) as in lse_merge (tc_logits.cu).  A sum that is not a normal,
// finite float well above the underflow range sets *bad (exact online-max path runs).
__device__ __forceinline__ void stats_finalize(float t, int i, float* __restrict__ lse, float* __restrict__ fac,
                                               int* __restrict__ fac_ok, int* __restrict__ bad, float c0, float c1,
                                               cudaGraphConditionalHandle cond) {
  if (!(t >= 0x1p-100f) || !isfinite(t)) {
    atomicExch(bad, 1);
    if (cond != 0) cudaGraphSetConditional(cond, 1);   // graph: run the exact statistics node
  }
  const float l2 = log2f(t);
  lse[i] = l2 * fs::kLn2;
  const bool ok = l2 > -120.f && l2 < 120.f;
  fac[i] = ok ? exp2f(-l2) * fmaf(c1, l2 * fs::kLn2, c0) : 0.f;
  if (!ok) *fac_ok = 0;
}

// Blocks [0, nrb): 256 rows each, the S column-chunk partials of a row summed by one thread.
// Blocks [nrb, ..): 32 columns each; the R row-block partials of a column are split over 8
// thread groups (fixed order: group q sums blocks q, q + 8, ...; the 8 group sums are then
// added in group order), so each thread has R / 8 loads in flight instead of R in sequence.
__global__ void __launch_bounds__(256) stats_merge_kernel(
    const float* __restrict__ part_rs, int S, int Na, const float* __restrict__ colpart, int R, int ldc, int Nb,
    float* __restrict__ lse_row, float* __restrict__ fac_row, float* __restrict__ lse_col, float* __restrict__ fac_col,
    int* __restrict__ fac_ok, int* __restrict__ bad, float rc0, float rc1, float cc0, float cc1, int force_bad,
    cudaGraphConditionalHandle cond, int nrb, float* __restrict__ colsum) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  if (force_bad && blockIdx.x == 0 && threadIdx.x == 0) {   // CRL_FORCE_STATS_FALLBACK (tests)
    atomicExch(bad, 1);
    if (cond != 0) cudaGraphSetConditional(cond, 1);
  }
  if ((int)blockIdx.x < nrb) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= Na) return;
    float t = 0.f;
    for (int s = 0; s < S; ++s) t += part_rs[(size_t)s * Na + i];
    stats_finalize(t, i, lse_row, fac_row, fac_ok, bad, rc0, rc1, cond);
    return;
  }
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int j = ((int)blockIdx.x - nrb) * 32 + c;
  float t = 0.f;
  if (j < Nb) {
#pragma unroll 4
    for (int s = q; s < R; s += 8) t += colpart[(size_t)s * ldc + j];
  }
  red[q][c] = t;
  __syncthreads();
  if (q == 0 && j < Nb) {
    float u = red[0][c];
#pragma unroll
    for (int k = 1; k < 8; ++k) u += red[k][c];
    // W > 1: this rank's rows only -> the column-sum all-reduce, then stats_col_finalize
    if (colsum != nullptr) colsum[j] = u;
    else stats_finalize(u, j, lse_col, fac_col, fac_ok, bad, cc0, cc1, cond);
  }
}

// W > 1: column sums over ALL ranks' rows (after the all-reduce) -> LSE' and
// factors of this rank's columns [col0, col0 + n)
__global__ void stats_col_finalize_kernel(const float* __restrict__ colsum, int col0, int n, float* __restrict__ lse_col,
                                          float* __restrict__ fac_col, int* __restrict__ fac_ok, int* __restrict__ bad,
                                          float cc0, float cc1) {
  pdl_wait();
  pdl_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) stats_finalize(colsum[col0 + i], i, lse_col, fac_col, fac_ok, bad, cc0, cc1, 0);
}

// ------------------------------------------------------------------------------- host side
bool tc_stats_supports(int D, int energy) {
  return (D == 64 || D == 128 || D == 256) &&
         (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_L2SQ || energy == CRL_ENERGY_COS);
}

// Column chunks per row block: enough work units to balance the persistent grid (~8 per SM)
// without units shorter than 2 tiles; at most 16 (row-sum partials per row).
int tc_stats_splits(int Na, int Nb, int num_sms) {
  const int rb = (Na + 127) / 128;
  const int tiles = (Nb + 127) / 128;
  int ch = 1;
  while (ch < 16 && ch * 2 <= tiles && (long)rb * ch < 8L * num_sms) ch *= 2;
  return ch;
}

static int g_stats_sms = 148;

template <int D, int ENERGY>
static cudaError_t launch_st(const CUtensorMap& a, const CUtensorMap& b, const TcStatsArgs& p, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = StCfg<D>::smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_stats_kernel<D, ENERGY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_stats_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  dim3 grid(min(p.n_units, g_stats_sms));
  return launch_pdl(tc_stats_kernel<D, ENERGY>, grid, dim3(128 + 128 * kStNWG), smem, st, a, b, p);
}

// One fused statistics pass + merge.  mA/mB: the logits operand maps (A box {64,128},
// B box {64,128}: tc_logits_maps with D <= 128).  part_rs [S][Na] (S = tc_stats_splits),
// colpart [R][ldc].
cudaError_t tc_stats_fused(int D, int energy, const CUtensorMap& mA, const CUtensorMap& mB, int Na, int Nb,
                           const float* a_stat, const float* b_stat, int S, float* part_rs, float* colpart, int ldc,
                           float* lse_row, float* fac_row, float* lse_col, float* fac_col, int* fac_ok, int* bad,
                           float rc0, float rc1, float cc0, float cc1, cudaGraphConditionalHandle cond,
                           cudaStream_t st, float* colsum) {
  TcStatsArgs p{};
  p.Na = Na; p.Nb = Nb;
  const int tiles = (Nb + 127) / 128;
  p.n_chunks = S;
  p.tiles_per_chunk = (tiles + S - 1) / S;
  p.n_units = ((Na + 127) / 128) * S;
  p.a_stat = a_stat; p.b_stat = b_stat; p.part_rs = part_rs; p.colpart = colpart; p.ldc = ldc;
  p.trace = std::getenv("CRL_STATS_TRACE") ? 1 : 0;
  cudaError_t e;
#define CRL_ST_DISPATCH(DD)                                                                                  \
  e = energy == CRL_ENERGY_L2     ? launch_st<DD, CRL_ENERGY_L2>(mA, mB, p, st)                             \
      : energy == CRL_ENERGY_L2SQ ? launch_st<DD, CRL_ENERGY_L2SQ>(mA, mB, p, st)                           \
                                  : launch_st<DD, CRL_ENERGY_COS>(mA, mB, p, st);
  if (D == 64) { CRL_ST_DISPATCH(64) }
  else if (D == 128) { CRL_ST_DISPATCH(128) }
  else if (D == 256) { CRL_ST_DISPATCH(256) }
#undef CRL_ST_DISPATCH
  else return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  const int R = (Na + 127) / 128;
  const int nrb = (Na + 255) / 256, ncb = (Nb + 31) / 32;
  return launch_pdl(stats_merge_kernel, dim3(nrb + ncb), dim3(256), 0, st, (const float*)part_rs, S, Na,
                    (const float*)colpart, R, ldc, Nb, lse_row, fac_row, lse_col, fac_col, fac_ok, bad, rc0, rc1,
                    cc0, cc1, std::getenv("CRL_FORCE_STATS_FALLBACK") ? 1 : 0, cond, nrb, colsum);
}

cudaError_t tc_stats_col_finalize(const float* colsum, int col0, int n, float* lse_col, float* fac_col, int* fac_ok,
                                  int* bad, float cc0, float cc1, cudaStream_t st) {
  return launch_pdl(stats_col_finalize_kernel, dim3((n + 255) / 256), dim3(256), 0, st, colsum, col0, n, lse_col, fac_col,
                    fac_ok, bad, cc0, cc1);
}

}  // namespace tc
}  // namespace crl
