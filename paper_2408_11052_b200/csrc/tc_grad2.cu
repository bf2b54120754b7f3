// tc_grad2.cu — the logits gradient pass (A4) at D = 256 (configs[4]'s representation size):
// both sides in ONE persistent launch, dL/dl consumed in registers, dPhi / dPsi on tcgen05.
//
// Paper: energies App. A.2 P:607-617 (L2 sign per reading A-01), InfoNCE fwd/bwd/sym P:619-630
// and the logsumexp penalty P:361 / Alg. 1 P:1052 (readings A-02..A-05).  The gradient of C4,
//   g_ij = (1/N)[c_r (p_ij - d_ij) + c_c (q_ij - d_ij)] + (2 beta / N) LSE_i p_ij,
// is mapped through the energy's VJP (C5: L2 w_ij = g_ij / r_ij, cos w_ij = g_ij / |b_j|) and
// contracted on the tensor core: dA_i = sum_j w_ij B_j (the L2 "- (sum_j w_ij) A_i" term, the
// positive pair and the cos projection are applied by grad_merge, tc_merge.cuh).
//   side 0: rows A = Phi (local), columns B = Psi (global)  -> dPhi
//   side 1: rows A = Psi (local), columns B = Phi (global)  -> dPsi   (coefficients swapped)
//
// Schedule (why it differs from tc_logits.cu's two-call GRAD kernel):
//  * One CTA per SM owns a CONTIGUOUS range of the linearised (side, row block, 128-column
//    tile) space (stream-K style): every CTA gets the same number of tiles +-1, a row block is
//    cut into at most two pieces, whose dA partials go to slot 0 (the piece holding the row
//    block's first tile) and slot 1 (the other piece, flagged for the merge).
//  * The 128 x 256 A tile of the current row block lives in TMEM (tcgen05.mma with an A
//    operand in tensor memory), so S = A B^T reads only B from SMEM.
//  * TMEM (512 columns): S 128 | dA accumulator 256 | A 128 (bf16 pairs).
//  * Per 128-column tile: S = A B^T (M 128, N 128, K 256: 16 MMAs) -> 8 epilogue warps (2
//    column halves x 4 lane quarters) form w_ij (one exp2 + one rsqrt / operand modifiers) as
//    a bf16 W tile in SMEM (SW128) -> dA += W B as two N = 128 halves (M 128, K 128: the same
//    SMEM B tile read as an MN-major operand).
//  * Why 128-column tiles (measured, scratch/g2_bench.cu + scratch/mma_bench.cu): the MMA
//    issuer returns only when its MMAs are nearly done, so every barrier wait of the issuing
//    thread is a tensor-pipe bubble; N = 64 S MMAs are also issue-bound (44 cycles vs the
//    32-cycle floor).  N = 128 S MMAs run at the 64-cycle floor and halve the waits per
//    column.  TMEM then holds one S buffer: the issuer puts S(t + 1) ahead of dA(t), so S(t + 1)
//    runs while the epilogue still works on tile t.
//  * B arrives as half tiles (D-chunks 2h, 2h + 1: 32 KB) in a 5-deep ring; dA's half h
//    releases half-slot h of its tile, so the next tile's loads start half a dA earlier.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_grad2.h"
#include "tc_pair.cuh"

namespace crl {
namespace tc {
namespace g2 {

constexpr int D = 256, BNT = 128, NH = 6;              // repr dim, tile columns, B half-tile ring
constexpr uint32_t CH_BYTES = BNT * 64 * 2;            // 16 KB: one D-chunk [128 j][64 D] (SW128)
constexpr uint32_t H_BYTES = 2 * CH_BYTES;             // 32 KB: half a B tile (D-chunks 2h, 2h + 1)
constexpr uint32_t W_BYTES = 128 * BNT * 2;            // 32 KB: W, two K-chunks [128 rows][64 j]
constexpr uint32_t STAT_FLOATS = 2 * BNT;              // b_stat, lcf of one tile (per warpgroup)
constexpr uint32_t BAR_BYTES = 256;
// 231,680 B of the 232,448 available: no alignment slack, the dynamic window must start on a
// 1 KB boundary (it does: the 1 KB system reservation precedes it; checked at run time)
constexpr size_t SMEM = NH * H_BYTES + W_BYTES + 2 * STAT_FLOATS * 4 + BAR_BYTES;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}
// 32 lanes x 32 bit, 32 consecutive columns per thread (registers -> TMEM)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// measurement: clock64 of pipeline events of CTA 0 (scratch/g2_bench.cu); no-op when null
__device__ __forceinline__ void g2_trace(unsigned long long* tr, int g, int ev) {
  if (tr != nullptr && blockIdx.x == 0 && g < 1024) tr[g * 8 + ev] = clock64();
}

// Per-row constants of a unit (row i of this side's A): log2-unit folds of the fast path.
// fac_fast: q_ij = p_ij 2^lse2_i 2^-lse2'_j, i.e. one MUFU op per logit for both softmaxes.
template <int ENERGY>
struct RowConst {
  float astat, lr2, Ei, Arow, cc0, cc1;
  f32x2 kL2, kM2, kA2, kLr2, kLrN2, kL1, kEi2, kAr2;
  __device__ __forceinline__ RowConst(const Grad2Side& sd, int row, bool rv, float invN, bool fac_fast) {
    constexpr float L2e2 = kLog2e * kLog2e;
    astat = rv ? sd.a_stat[row] : 0.f;
    const float lr_nat = rv ? sd.lr[row] : 0.f;
    lr2 = lr_nat * kLog2e;
    Ei = fac_fast ? ex2(lr2) : 0.f;
    Arow = invN * sd.c_r + 2.f * invN * sd.beta_r * lr_nat;
    cc0 = invN * sd.c_c;
    cc1 = 2.f * invN * sd.beta_c;
    // L2: x = d2 (log2 e)^2 (sqrt taken per logit); L2^2: x = d2 log2 e is the log2-unit logit
    constexpr float kx = ENERGY == CRL_ENERGY_L2SQ ? kLog2e : L2e2;
    kL2 = f2_pack(kx, kx);
    kM2 = f2_pack(-2.f * kx, -2.f * kx);
    const float ka = ENERGY == CRL_ENERGY_L2 ? astat * L2e2 : astat * kLog2e;
    kA2 = f2_pack(ka, ka);
    kLr2 = f2_pack(lr2, lr2);
    kLrN2 = f2_pack(-lr2, -lr2);
    kL1 = f2_pack(kLog2e, kLog2e);
    // L2: w = g rs' log2e;  L2^2: w = 2 g (dl/dphi = -2 (phi - psi))
    const float fe = ENERGY == CRL_ENERGY_L2 ? kLog2e : (ENERGY == CRL_ENERGY_L2SQ ? 2.f : 1.f);
    kEi2 = f2_pack(Ei * fe, Ei * fe);
    kAr2 = f2_pack(Arow * fe, Arow * fe);
  }
};

// w_ij of one row for NC columns c0 .. c0 + NC - 1 of a 128-column tile -> NC / 2 bf16 pairs; the L2
// row sum of w accumulates into wsum.  raw: S_ij (fp32 bits); bst: [b_stat 128][lcf 128] of the
// tile in SMEM; lc_tile: the column LSEs of the tile in global memory (exact-q path only).
// of every 4 logit pairs of the fast path, this many take exp2 on the FMA / ALU pipes
// (ex2_pair_fma, tc_common.cuh) instead of the MUFU (measured on B200, netscale pair pass:
// 0 -> 432 us, 1 -> 436, 2 -> 447: the epilogue is latency- rather than XU-bound)
#ifndef CRL_G2_EMU
#define CRL_G2_EMU 0
#endif
constexpr int kG2EmuPairs = CRL_G2_EMU;
constexpr int kG2RsqPairs = 0;                         // default of CRL_G2_RSQ (tc_grad2p, L2)

// rsqrt on the FMA pipe for a pair (L2, RQ of every 4 pairs): exponent-halving integer guess,
// two Newton steps y <- y (3/2 - (x/2) y^2) in packed FFMA2 / FMUL2 (relative error ~5e-6)
__device__ __forceinline__ f32x2 rsq_pair_fma(float x0, float x1) {
  int i0, i1;
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i0) : "r"(__float_as_int(x0)), "r"((int)0x80000000), "r"(0x5f375a86));
  asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(i1) : "r"(__float_as_int(x1)), "r"((int)0x80000000), "r"(0x5f375a86));
  const f32x2 nhx = f2_mul(f2_pack(x0, x1), f2_pack(-0.5f, -0.5f));
  f32x2 y = f2_pack(__int_as_float(i0), __int_as_float(i1));
#pragma unroll
  for (int it = 0; it < 2; ++it) y = f2_mul(y, f2_fma(f2_mul(nhx, y), y, f2_pack(1.5f, 1.5f)));
  return y;
}

template <int ENERGY, int NC, int RQ = 0>
__device__ __forceinline__ void w_tile(const uint32_t (&raw)[NC], const float* bst, int c0, int nval, bool fast,
                                       bool fac_fast, const RowConst<ENERGY>& k, const float* lc_tile,
                                       uint32_t (&pk)[NC / 2], float& wsum) {
  constexpr int BNT = 128;
  constexpr float kEpsL2e = kEpsL2 * kLog2e * kLog2e;
  constexpr bool DIFF = ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ;   // row sums of w needed
  if (fast) {
    // full tile, normal factors: packed fp32 pairs (FFMA2 / FMUL2 / FADD2), constants
    // folded into log2 units, column statistics by 16-byte loads; per logit 2 MUFU ops
    //   L2 : x = d2 (log2 e)^2, rs = 1/sqrt(x), s = x rs = r log2 e,
    //        p = 2^-(s + lse2_i), w = p (Ei lcf_j + A_i) log2e rs = g_ij / r_ij
    //   L2^2: x = d2 log2 e, p = 2^-(x + lse2_i), w = p (Ei lcf_j + A_i) 2 = 2 g_ij
    //   cos: p = 2^(v a_i b_j log2 e - lse2_i), w = p (Ei lcf_j + A_i) b_j
    //   dot: p = 2^(v log2 e - lse2_i),         w = p (Ei lcf_j + A_i)
    f32x2 ws2 = f2_pack(0.f, 0.f);
#pragma unroll
    for (int i4 = 0; i4 < NC / 4; ++i4) {
      const float4 bs = lds_f4(smem_u32(bst + c0 + 4 * i4));
      const float4 lf = lds_f4(smem_u32(bst + BNT + c0 + 4 * i4));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 4 * i4 + 2 * h;
        const f32x2 v2 = f2_pack(__uint_as_float(raw[i]), __uint_as_float(raw[i + 1]));
        const f32x2 b2 = h ? f2_pack(bs.z, bs.w) : f2_pack(bs.x, bs.y);
        const f32x2 l2 = h ? f2_pack(lf.z, lf.w) : f2_pack(lf.x, lf.y);
        const f32x2 fct = f2_fma(k.kEi2, l2, k.kAr2);
        float p0, p1, w0, w1;
        if (ENERGY == CRL_ENERGY_L2) {
          float x0, x1;
          f2_unpack(f2_fma(k.kM2, v2, f2_fma(k.kL2, b2, k.kA2)), x0, x1);
          x0 = fmaxf(x0, kEpsL2e); x1 = fmaxf(x1, kEpsL2e);
          const f32x2 rs2 = ((2 * i4 + h) & 3) < RQ ? rsq_pair_fma(x0, x1) : f2_pack(rsq(x0), rsq(x1));
          float a0, a1;
          f2_unpack(f2_fma(f2_pack(x0, x1), rs2, k.kLr2), a0, a1);
          if (((2 * i4 + h) & 3) < kG2EmuPairs) ex2_pair_fma(-a0, -a1, p0, p1);
          else { p0 = ex2_neg(a0); p1 = ex2_neg(a1); }
          f2_unpack(f2_mul(f2_mul(f2_pack(p0, p1), fct), rs2), w0, w1);
        } else if (ENERGY == CRL_ENERGY_L2SQ) {
          float x0, x1, a0, a1;
          f2_unpack(f2_fma(k.kM2, v2, f2_fma(k.kL2, b2, k.kA2)), x0, x1);
          f2_unpack(f2_add(f2_pack(fmaxf(x0, 0.f), fmaxf(x1, 0.f)), k.kLr2), a0, a1);
          if (((2 * i4 + h) & 3) < kG2EmuPairs) ex2_pair_fma(-a0, -a1, p0, p1);
          else { p0 = ex2_neg(a0); p1 = ex2_neg(a1); }
          f2_unpack(f2_mul(f2_pack(p0, p1), fct), w0, w1);
        } else if (ENERGY == CRL_ENERGY_COS) {
          float a0, a1;
          f2_unpack(f2_fma(f2_mul(v2, b2), k.kA2, k.kLrN2), a0, a1);
          if (((2 * i4 + h) & 3) < kG2EmuPairs) ex2_pair_fma(a0, a1, p0, p1);
          else { p0 = ex2(a0); p1 = ex2(a1); }
          f2_unpack(f2_mul(f2_mul(f2_pack(p0, p1), fct), b2), w0, w1);
        } else {
          float a0, a1;
          f2_unpack(f2_fma(v2, k.kL1, k.kLrN2), a0, a1);
          if (((2 * i4 + h) & 3) < kG2EmuPairs) ex2_pair_fma(a0, a1, p0, p1);
          else { p0 = ex2(a0); p1 = ex2(a1); }
          f2_unpack(f2_mul(f2_pack(p0, p1), fct), w0, w1);
        }
        pk[i >> 1] = pack_bf16x2(w0, w1);
        if (DIFF) ws2 = f2_add(ws2, f2_pack(w0, w1));
      }
    }
    if (DIFF) {
      float s0, s1;
      f2_unpack(ws2, s0, s1);
      wsum += s0 + s1;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NC; i += 2) {
      float wv2[2];
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const int jl = c0 + i + e2;
        const float v = __uint_as_float(raw[i + e2]);
        const bool cv = jl < nval;
        const float bj = bst[jl];
        float l, rs = 0.f;
        if (ENERGY == CRL_ENERGY_L2) {
          const float d2 = fmaxf(fmaf(-2.f, v, k.astat + bj), 0.f) + kEpsL2;
          rs = rsq(d2);
          l = -d2 * rs;
        } else if (ENERGY == CRL_ENERGY_L2SQ) {
          l = -fmaxf(fmaf(-2.f, v, k.astat + bj), 0.f);
        } else if (ENERGY == CRL_ENERGY_COS) {
          l = v * k.astat * bj;
        } else {
          l = v;
        }
        const float tv = cv ? l * kLog2e : -INFINITY;
        const float pe = ex2(tv - k.lr2);
        float gij;
        if (fac_fast) {
          gij = pe * fmaf(k.Ei, bst[BNT + jl], k.Arow);
        } else {
          const float lc = cv ? __ldg(lc_tile + jl) : 0.f;
          const float qe = ex2(tv - lc * kLog2e);
          gij = fmaf(pe, k.Arow, qe * fmaf(k.cc1, lc, k.cc0));
        }
        float wv;
        if (ENERGY == CRL_ENERGY_L2) wv = gij * rs;
        else if (ENERGY == CRL_ENERGY_L2SQ) wv = 2.f * gij;
        else if (ENERGY == CRL_ENERGY_COS) wv = gij * bj;
        else wv = gij;
        wv = cv ? wv : 0.f;                               // padded columns: no NaN from pad stats
        if (DIFF) wsum += wv;
        wv2[e2] = wv;
      }
      pk[i >> 1] = pack_bf16x2(wv2[0], wv2[1]);
    }
  }
}

// the tile range of CTA c of G over X tiles: [start(c), start(c + 1))
__host__ __device__ __forceinline__ long range_start(long c, long X, long G) { return (c * X) / G; }

}  // namespace g2

template <int ENERGY>
__global__ void __launch_bounds__(352, 1) tc_grad2_kernel(const __grid_constant__ CUtensorMap tmB0,
                                                          const __grid_constant__ CUtensorMap tmB1, const Grad2Args p) {
  using namespace g2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sB = smem_raw;                                                 // [NH] B half tiles
  uint8_t* sW = sB + NH * H_BYTES;                                        // W tile
  float* sStat = reinterpret_cast<float*>(sW + W_BYTES);                  // [2 warpgroups][2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStat + 2 * STAT_FLOATS);
  uint64_t* h_full = bars;                 // [NH]  half tile landed
  uint64_t* h_empty = h_full + NH;         // [NH]  half tile consumed by its dA
  uint64_t* st_full = h_empty + NH;        // [2]   column statistics of tile g (slot g & 1) landed
  uint64_t* st_empty = st_full + 2;        // [2]   ... consumed
  uint64_t* s_full = st_empty + 2;         //       S of the current tile is in TMEM
  uint64_t* s_empty = s_full + 1;          //       S has been loaded (the single S buffer is free)
  uint64_t* w_full = s_empty + 1;          //       W of the current tile is in SMEM
  uint64_t* w_empty = w_full + 1;          //       dA of the current tile has read W
  uint64_t* a_full = w_empty + 1;          //       A of the current unit is in TMEM
  uint64_t* da_full = a_full + 1;          //       the unit's dA accumulation is complete
  uint64_t* da_empty = da_full + 1;        //       the unit's dA has been read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(da_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long X = 2L * p.RB * p.TPB;
  const long x0 = range_start(blockIdx.x, X, gridDim.x), x1 = range_start(blockIdx.x + 1, X, gridDim.x);
  // unit = the maximal run of this CTA's tiles inside one (side, row block)
  auto unit_at = [&](long x, int& side, int& rb, int& tb, int& nt) {
    const long r = x / p.TPB;
    tb = (int)(x - r * p.TPB);
    side = (int)(r / p.RB);
    rb = (int)(r - (long)side * p.RB);
    nt = (int)min((long)(p.TPB - tb), x1 - x);
  };

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();     // SW128 operands need 1 KB alignment
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmB1);
    for (int s = 0; s < NH; ++s) { mbar_init(&h_full[s], 1); mbar_init(&h_empty[s], 1); }
    for (int e = 0; e < 2; ++e) { mbar_init(&st_full[e], 1); mbar_init(&st_empty[e], 8); }
    mbar_init(s_full, 1); mbar_init(s_empty, 8);
    mbar_init(w_full, 8); mbar_init(w_empty, 1);
    mbar_init(a_full, 8); mbar_init(da_full, 1); mbar_init(da_empty, 8);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_s = tmem;
  const uint32_t tm_da = tmem + 128;
  const uint32_t tm_a = tmem + 384;
  pdl_wait();
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      int g = 0;
      for (long x = x0; x < x1;) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        const CUtensorMap* mB = side ? &tmB1 : &tmB0;
        for (int t = 0; t < nt; ++t, ++g) {
          const int j0 = (tb + t) * BNT;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int u = 2 * g + h, hs = u % NH;
            mbar_wait(&h_empty[hs], ((u / NH) & 1) ^ 1);
            g2_trace(p.trace, g, h);
            if (p.dbg & 16) { mbar_arrive(&h_full[hs]); continue; }
            mbar_expect_tx(&h_full[hs], H_BYTES);
            uint8_t* dst = sB + hs * H_BYTES;
            tma_load_2d(dst, mB, &h_full[hs], 64 * (2 * h), j0);            // B {D, rows} box {64, 128}
            tma_load_2d(dst + CH_BYTES, mB, &h_full[hs], 64 * (2 * h + 1), j0);
          }
        }
        x += nt;
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {
      // ---------------------------------------------------------------- column statistics
      // (their own producer: a slot is free only once the epilogue is done with it, which
      // must not hold back the B stream)
      int g = 0;
      for (long x = x0; x < x1;) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        const Grad2Side& sd = p.side[side];
        for (int t = 0; t < nt; ++t, ++g) {
          const int j0 = (tb + t) * BNT;
          const int e = g & 1;
          mbar_wait(&st_empty[e], ((g >> 1) & 1) ^ 1);
          mbar_expect_tx(&st_full[e], STAT_FLOATS * 4);
          float* st = sStat + e * STAT_FLOATS;
          bulk_g2s(st, sd.b_stat + j0, BNT * 4, &st_full[e]);
          bulk_g2s(st + BNT, sd.lcf + j0, BNT * 4, &st_full[e]);
        }
        x += nt;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t id_s = idesc_bf16_f32(128, BNT, false, false);
      const uint32_t id_da = idesc_bf16_f32(128, D, false, true);
      auto issue_s = [&](int g) {
        mbar_wait(s_empty, (g & 1) ^ 1);                  // S(g - 1) has been loaded
        mbar_wait(&h_full[(2 * g) % NH], ((2 * g) / NH) & 1);
        mbar_wait(&h_full[(2 * g + 1) % NH], ((2 * g + 1) / NH) & 1);
        tc_fence_after();
        if (!(p.dbg & 4)) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            const uint32_t cb = smem_u32(sB + ((2 * g + (c >> 1)) % NH) * H_BYTES + (c & 1) * CH_BYTES);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              mma_ts(tm_s, tm_a + (uint32_t)(8 * (4 * c + ks)), smem_desc_sw128(cb + ks * 32, 16, 1024), id_s,
                     (c | ks) != 0);
          }
        }
        mma_commit(s_full);
        g2_trace(p.trace, g, 2);
      };
      auto issue_da = [&](int g, bool first, int k) {
        if (first) {
          mbar_wait(da_empty, (k & 1) ^ 1);               // unit k - 1's dA has been read out
          tc_fence_after();
        }
        mbar_wait(w_full, g & 1);
        tc_fence_after();
        const int hs0 = (2 * g) % NH;                     // NH even: the halves are adjacent slots
        if (!(p.dbg & 2)) {
          const uint32_t w_base = smem_u32(sW), b0 = smem_u32(sB + hs0 * H_BYTES);
#pragma unroll
          for (int ks = 0; ks < BNT / 16; ++ks)          // K = the 128 columns of the tile, N = D
            mma_bf16(tm_da, smem_desc_sw128(w_base + (ks >> 2) * CH_BYTES + (ks & 3) * 32, 16, 1024),
                     smem_desc_sw128(b0 + ks * 2048, CH_BYTES, 1024), id_da, !(first && ks == 0));
        }
        mma_commit(&h_empty[hs0]);
        mma_commit(&h_empty[hs0 + 1]);
        mma_commit(w_empty);
        g2_trace(p.trace, g, 3);
      };
      // S(t + 1) is issued ahead of dA(t): it needs only the epilogue's TMEM load of S(t), while
      // dA(t) needs the whole W(t), so S(t + 1) runs under tile t's epilogue.  Six half-tile
      // slots: B(t + 2) streams in while B(t) and B(t + 1) are still referenced.
      int g = 0, k = 0;
      for (long x = x0; x < x1; ++k) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        mbar_wait(a_full, k & 1);                          // A of this unit in TMEM
        tc_fence_after();
        issue_s(g);
        for (int t = 0; t < nt; ++t) {
          if (t + 1 < nt) issue_s(g + t + 1);
          issue_da(g + t, t == 0, k);
        }
        mma_commit(da_full);
        g += nt;
        x += nt;
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..9)
    // Thread = row r of the row block (TMEM lane); warpgroup wg takes columns 64 wg .. + 63
    // of every tile (W K-chunk wg), the K half wg of A and the D half wg of dA.
    const int wg = (warp - 2) >> 2;
    const int q = warp & 3;                               // TMEM lane quarter
    const int r = q * 32 + lane;                          // row within the row block
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool tr_lead = p.trace != nullptr && warp == 2 && lane == 0;
    const bool fac_fast = *p.fac_ok != 0;
    const int c0 = 64 * wg;
    int g = 0, k = 0;
    int prev_side = 0, prev_rb = 0, prev_slot = 0;
    auto readout = [&](int side, int rb, int slot, int kk) {
      // dA of unit kk: row r, D half wg -> part_da[slot]
      mbar_wait(da_full, kk & 1);
      tc_fence_after();
      const int row = rb * 128 + r;
      const Grad2Side& sd = p.side[side];
      const bool rv = row < p.Na;
      float* out = sd.part_da + ((size_t)slot * p.Na + row) * D + 128 * wg;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32_nowait(tm_da + lane_off + 128 * wg + 32 * c, v);
        tmem_ld_wait();
        if (rv) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(out + 32 * c)[i] =
                make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                            __uint_as_float(v[4 * i + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(da_empty);
    };
    for (long x = x0; x < x1; ++k) {
      int side, rb, tb, nt;
      unit_at(x, side, rb, tb, nt);
      const Grad2Side& sd = p.side[side];
      const int row = rb * 128 + r;
      const bool rv = row < p.Na;
      // ---- A of this row block -> TMEM (the previous unit's S MMAs are complete: its last
      // tile's S was consumed below).  Row r, K half wg: 128 bf16 = 64 packed 32-bit columns.
      {
        uint32_t av[64];
        if (rv) {
          const uint4* src = reinterpret_cast<const uint4*>(sd.A + (size_t)row * D + 128 * wg);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint4 u = __ldg(src + i);
            av[4 * i] = u.x; av[4 * i + 1] = u.y; av[4 * i + 2] = u.z; av[4 * i + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) av[i] = 0u;
        }
        tmem_st32(tm_a + lane_off + 64 * wg, *reinterpret_cast<uint32_t(*)[32]>(av));
        tmem_st32(tm_a + lane_off + 64 * wg + 32, *reinterpret_cast<uint32_t(*)[32]>(av + 32));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full);
      }
      if (k > 0) readout(prev_side, prev_rb, prev_slot, k - 1);
      const RowConst<ENERGY> kc(sd, row, rv, p.invN, fac_fast);
      float wsum = 0.f;
      for (int t = 0; t < nt; ++t, ++g) {
        const int sl = g & 1;
        const int j0 = (tb + t) * BNT;
        const int nval = p.Nb - j0;                       // valid columns of this tile (>= 1)
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        if (tr_lead) g2_trace(p.trace, g, 4);
        uint32_t raw[64];
        if (p.dbg & 8) {
#pragma unroll
          for (int i = 0; i < 64; ++i) raw[i] = __float_as_uint(1.f + i + r);
        } else {
          tmem_ld32_nowait(tm_s + lane_off + c0, *reinterpret_cast<uint32_t(*)[32]>(raw));
          tmem_ld32_nowait(tm_s + lane_off + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
          tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty);
        if (tr_lead) g2_trace(p.trace, g, 5);
        mbar_wait(&st_full[sl], (g >> 1) & 1);
        const float* bst = sStat + sl * STAT_FLOATS;     // [b_stat 128][lcf 128]
        const bool fast = fac_fast && nval >= BNT && !(p.dbg & 1);
        uint32_t pk[32];                                  // bf16 pairs of w, row r, 64 columns
        if (p.dbg & 1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = raw[2 * i] ^ raw[2 * i + 1];
        } else {
          w_tile<ENERGY, 64>(raw, bst, c0, nval, fast, fac_fast, kc, sd.lc + j0, pk, wsum);
        }
        if (tr_lead) g2_trace(p.trace, g, 6);
        if (g >= 1) mbar_wait(w_empty, (g - 1) & 1);      // dA(g - 1) has read W
        const uint32_t wt = smem_u32(sW + wg * CH_BYTES);  // K-chunk wg = this warp's 64 columns
#pragma unroll
        for (int u = 0; u < 8; ++u)
          sts_u4(wt + sw128_off(r, 8 * u), make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) { mbar_arrive(w_full); mbar_arrive(&st_empty[sl]); }
        if (tr_lead) g2_trace(p.trace, g, 7);
      }
      // this warpgroup's share of the L2 row sums of the unit ("- (sum_j w_ij) A_i" term of
      // the merge): sub-slot wg of the unit's partial slot
      const int slot = tb == 0 ? 0 : 1;
      if ((ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) && rv)
        sd.part_rs[((size_t)(2 * slot + wg)) * p.Na + row] = wsum;
      prev_side = side; prev_rb = rb; prev_slot = slot;
      x += nt;
    }
    if (k > 0) readout(prev_side, prev_rb, prev_slot, k - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =============================================================================== CTA pairs
// tc_grad2p: the same pass on CTA PAIRS (tcgen05 cta_group::2).  A pair owns 256 rows of a side
// (CTA r: rows [128 r, 128 r + 128) of the row-block pair, its 128 A rows TMA-loaded into its own
// SMEM once per unit) and walks 128-column tiles:
//   S   = A B^T   M 256, N 128, K 256: rank r stages the B tile's rows [64 r, 64 r + 64)
//                 (all 256 D: the "S part", 32 KB); S double-buffered in TMEM (2 x 128 columns)
//   dA += W B     M 256, N 256, K 128: rank r stages the B tile's D half [128 r, 128 r + 128)
//                 (all 128 rows: the "dA part", 32 KB) and its own W rows (one W buffer)
// so each SM reads half of each B operand from SMEM.  TMEM: S[2] 256 + dA 256 = 512 columns.
// Two producers: warp 0 (A rows, S parts) and the statistics warp (column statistics, dA parts),
// so an S part runs two tiles ahead of the dA part of the same tile.
// Epilogue, W tile and per-row constants exactly as tc_grad2 (w_tile).
// Measured on B200 (scratch/g2_bench.cu, netscale 16384 x 16384 x 256, L2, 221 tiles per pair):
// 420 us; the previous layout (A in TMEM, one S buffer) 423 us; no MMAs at all 345 us, no MMA and
// no epilogue math 177 us.  The epilogue (about 14 instructions and 4 MUFU ops per logit pair)
// bounds the pass; moving rsqrt to the FMA pipe (CRL_G2_RSQ = 1..4 of every 4 pairs) costs
// 435 / 453 / 481 / 522 us, so the MUFU is not the binding unit.
namespace g2p {
constexpr int D = 256, BNT = 128, NS = 2, ND = 2;
#ifndef CRL_G2P_NWG
#define CRL_G2P_NWG 4
#endif
constexpr int kNWG = CRL_G2P_NWG;                      // epilogue warpgroups (2 or 4)
constexpr uint32_t SP_CH = 64 * 128;                   // 8 KB: [64 rows][64 D] (SW128)
constexpr uint32_t SP_BYTES = 4 * SP_CH;               // 32 KB: S part
constexpr uint32_t DP_CH = BNT * 128;                  // 16 KB: [128 rows][64 D]
constexpr uint32_t DP_BYTES = 2 * DP_CH;               // 32 KB: dA part
constexpr uint32_t W_CH = 128 * 128;                   // 16 KB: W K-chunk [128 rows][64 j]
constexpr uint32_t W_BYTES = 2 * W_CH;                 // the W tile (single: dA(t - 1) has read it long before
                                                       // W(t) is written, one epilogue math phase later)
constexpr uint32_t A_CH = 128 * 128;                   // 16 KB: A K-chunk [128 rows][64 D]
constexpr uint32_t A_BYTES = 4 * A_CH;                 // 64 KB: this CTA's 128 A rows (SMEM operand of S)
constexpr uint32_t STAT_FLOATS = 2 * BNT;
constexpr size_t SMEM = A_BYTES + NS * SP_BYTES + ND * DP_BYTES + W_BYTES + 2 * STAT_FLOATS * 4 + 256;
}  // namespace g2p

template <int ENERGY, int RQ>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 128 * g2p::kNWG, 1)
    tc_grad2p_kernel(const __grid_constant__ CUtensorMap tmD0, const __grid_constant__ CUtensorMap tmD1,
                     const __grid_constant__ CUtensorMap tmS0, const __grid_constant__ CUtensorMap tmS1,
                     const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                     const __grid_constant__ CUtensorMap tmW, const Grad2Args p) {
  using namespace g2p;
  using namespace pair;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sA = smem_raw;                                                 // A rows of the unit
  uint8_t* sS = sA + A_BYTES;                                             // [NS] S parts
  uint8_t* sD = sS + NS * SP_BYTES;                                       // [ND] dA parts
  uint8_t* sW = sD + ND * DP_BYTES;                                       // W tile
  float* sStat = reinterpret_cast<float*>(sW + W_BYTES);                  // [2][b_stat 128, lcf 128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStat + 2 * STAT_FLOATS);
  uint64_t* sp_full = bars;                // [NS] leader: both CTAs' S-part bytes
  uint64_t* sp_free = sp_full + NS;        // [NS] both: S MMA done (multicast)
  uint64_t* dp_full = sp_free + NS;        // [ND] leader: both CTAs' dA-part bytes
  uint64_t* dp_free = dp_full + ND;        // [ND] both: dA MMA done
  uint64_t* st_full = dp_free + ND;        // [2] local column statistics
  uint64_t* st_empty = st_full + 2;        // [2]
  uint64_t* s_full = st_empty + 2;         // [2] both: S accumulator b ready
  uint64_t* s_empty = s_full + 2;          // [2] leader: every epilogue warp loaded S accumulator b
  uint64_t* w_full = s_empty + 2;          // leader: every epilogue warp wrote W
  uint64_t* w_empty = w_full + 1;          // both: the dA MMA read W
  uint64_t* a_full = w_empty + 1;          // leader: both CTAs' A rows of the unit landed (TMA)
  uint64_t* a_empty = a_full + 1;          // both: the unit's last S MMA completed
  uint64_t* da_full = a_empty + 1;         // both: the unit's dA complete
  uint64_t* da_empty = da_full + 1;        // leader: dA read out
  uint64_t* w_loc = da_empty + 1;          // local: every epilogue warp of this CTA wrote W (w_store)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_loc + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const long X = (long)(p.nsides == 1 ? 1 : 2) * p.RB * p.TPB;           // p.RB: row-block PAIRS
  const bool wst = p.w_store != 0;                                        // (host: only with nsides = 1)
  const long x0 = g2::range_start(cid, X, ncl), x1 = g2::range_start(cid + 1, X, ncl);
  auto unit_at = [&](long x, int& side, int& rb, int& tb, int& nt) {
    const long r = x / p.TPB;
    tb = (int)(x - r * p.TPB);
    side = (int)(r / p.RB);
    rb = (int)(r - (long)side * p.RB);
    nt = (int)min((long)(p.TPB - tb), x1 - x);
  };

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();
    tma_prefetch_desc(&tmD0); tma_prefetch_desc(&tmD1);
    tma_prefetch_desc(&tmS0); tma_prefetch_desc(&tmS1);
    tma_prefetch_desc(&tmA0); tma_prefetch_desc(&tmA1);
    if (wst) tma_prefetch_desc(&tmW);
    for (int i = 0; i < NS; ++i) { mbar_init(&sp_full[i], 1); mbar_init(&sp_free[i], 1); }
    for (int i = 0; i < ND; ++i) { mbar_init(&dp_full[i], 1); mbar_init(&dp_free[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&st_full[i], 1); mbar_init(&st_empty[i], 4 * kNWG); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8 * kNWG); }
    mbar_init(w_full, 8 * kNWG); mbar_init(w_empty, wst ? 2 : 1);   // dA MMA (+ the W store) read W
    mbar_init(a_full, 1); mbar_init(a_empty, 1);
    mbar_init(da_full, 1); mbar_init(da_empty, 8 * kNWG);
    mbar_init(w_loc, 4 * kNWG);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_s = tmem, tm_da = tmem + 256;       // S double buffer [2][128 cols], dA [256 cols]
  pdl_wait();
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer (both)
      int g = 0, k = 0;
      const uint32_t afb = mapa(smem_u32(a_full), 0);
      for (long x = x0; x < x1; ++k) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        const CUtensorMap* mS = side ? &tmS1 : &tmS0;
        // the unit's A rows (zero-filled past the batch): after the previous unit's last S MMA
        mbar_wait(a_empty, (k & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(a_full, 2 * A_BYTES);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tma_load_2d_pair(smem_u32(sA + c * A_CH), side ? &tmA1 : &tmA0, afb, 64 * c, rb * 256 + 128 * (int)rank);
        for (int t = 0; t < nt; ++t, ++g) {
          const int j0 = (tb + t) * BNT;
          const int ss = g % NS;
          mbar_wait(&sp_free[ss], ((g / NS) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&sp_full[ss], 2 * SP_BYTES);
          const uint32_t sfb = mapa(smem_u32(&sp_full[ss]), 0);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            tma_load_2d_pair(smem_u32(sS + ss * SP_BYTES + c * SP_CH), mS, sfb, 64 * c, j0 + 64 * (int)rank);
          g2::g2_trace(p.trace, g, 0);
        }
        x += nt;
      }
    }
  } else if (warp == 2 + 4 * kNWG) {
    if (lane == 0) {
      // ------------------------------------------ column statistics (local) + dA parts (both CTAs)
      // (the S parts and A rows have their own producer: an S part runs two tiles ahead of the
      // dA part of the same tile, whose slot frees only when dA(t - ND) completed)
      int g = 0;
      for (long x = x0; x < x1;) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        const Grad2Side& sd = p.side[side];
        const CUtensorMap* mD = side ? &tmD1 : &tmD0;
        for (int t = 0; t < nt; ++t, ++g) {
          const int j0 = (tb + t) * BNT;
          const int ds = g % ND;
          mbar_wait(&dp_free[ds], ((g / ND) & 1) ^ 1);
          g2::g2_trace(p.trace, g, 1);
          if (rank == 0) mbar_expect_tx(&dp_full[ds], 2 * DP_BYTES);
          const uint32_t dfb = mapa(smem_u32(&dp_full[ds]), 0);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_2d_pair(smem_u32(sD + ds * DP_BYTES + c * DP_CH), mD, dfb, 128 * (int)rank + 64 * c, j0);
          const int e = g & 1;
          mbar_wait(&st_empty[e], ((g >> 1) & 1) ^ 1);
          mbar_expect_tx(&st_full[e], STAT_FLOATS * 4);
          float* st = sStat + e * STAT_FLOATS;
          g2::bulk_g2s(st, sd.b_stat + j0, BNT * 4, &st_full[e]);
          g2::bulk_g2s(st + BNT, sd.lcf + j0, BNT * 4, &st_full[e]);
        }
        x += nt;
      }
    }
  } else if (warp == 3 + 4 * kNWG) {
    if (lane == 0 && wst) {
      // ------------------------------------------ W store (local): the tile's bf16 W -> global
      // (side 0 only; rows past Na / columns past Nb are clipped by the map or skipped whole)
      const int row0 = 128 * (int)rank;
      int g = 0;
      for (long x = x0; x < x1;) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        const int r0 = rb * 256 + row0;
        for (int t = 0; t < nt; ++t, ++g) {
          const int j0 = (tb + t) * BNT;
          mbar_wait(w_loc, g & 1);
          if (r0 < p.Na) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
              if (j0 + 64 * c < p.Nb && !(p.dbg & 8)) g2::tma_store_2d(&tmW, smem_u32(sW + c * W_CH), j0 + 64 * c, r0);
            g2::bulk_commit();
            g2::bulk_wait_read();
          }
          mbar_arrive(w_empty);                             // local: the tile may be overwritten
        }
        x += nt;
      }
      g2::bulk_wait_all();
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader)
      const uint32_t id_s = idesc_bf16_f32(256, BNT, false, false);
      const uint32_t id_da = idesc_bf16_f32(256, D, false, true);
      auto issue_s = [&](int g, bool last) {
        const int sb = g & 1;
        mbar_wait(&s_empty[sb], ((g >> 1) & 1) ^ 1);   // both CTAs loaded S(g - 2)
        const int ss = g % NS;
        mbar_wait(&sp_full[ss], (g / NS) & 1);
        tc_fence_after();
        if (!(p.dbg & 4))
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_pair(tm_s + 128u * (uint32_t)sb, smem_desc_sw128(smem_u32(sA + c * A_CH) + ks * 32, 16, 1024),
                     smem_desc_sw128(smem_u32(sS + ss * SP_BYTES + c * SP_CH) + ks * 32, 16, 1024), id_s,
                     (c | ks) != 0);
        commit_pair(&sp_free[ss]);
        commit_pair(&s_full[sb]);
        if (last) commit_pair(a_empty);        // the unit's A may be overwritten
        g2::g2_trace(p.trace, g, 2);
      };
      auto issue_da = [&](int g, bool first, int k) {
        if (first) {
          mbar_wait(da_empty, (k & 1) ^ 1);   // unit k - 1's dA read out (both)
          tc_fence_after();
        }
        mbar_wait(w_full, g & 1);
        const int ds = g % ND;
        mbar_wait(&dp_full[ds], (g / ND) & 1);
        tc_fence_after();
        const uint32_t w_base = smem_u32(sW), b0 = smem_u32(sD + ds * DP_BYTES);
        if (!(p.dbg & 2))
#pragma unroll
        for (int ks = 0; ks < BNT / 16; ++ks)            // K = the 128 rows of the tile
          mma_pair(tm_da, smem_desc_sw128(w_base + (ks >> 2) * W_CH + (ks & 3) * 32, 16, 1024),
                   smem_desc_sw128(b0 + ks * 2048, DP_CH, 1024), id_da, !(first && ks == 0));
        commit_pair(&dp_free[ds]);
        commit_pair(w_empty);
        g2::g2_trace(p.trace, g, 3);
      };
      int g = 0, k = 0;
      for (long x = x0; x < x1; ++k) {
        int side, rb, tb, nt;
        unit_at(x, side, rb, tb, nt);
        mbar_wait(a_full, k & 1);             // A of this unit in both CTAs' SMEM
        tc_fence_after();
        // S is double-buffered in TMEM and runs two tiles ahead of dA: S(t + 2) needs the TMEM
        // load of S(t) only (early in tile t's epilogue), so the S MMA and its commit latency
        // hide under the epilogue; dA(t) follows W(t) (S parts and dA parts have separate rings,
        // so the early S cannot wait on a slot only a later dA frees)
        issue_s(g, nt == 1);
        if (nt > 1) issue_s(g + 1, nt == 2);
        for (int t = 0; t < nt; ++t) {
          if (t + 2 < nt) issue_s(g + t + 2, t + 3 == nt);
          issue_da(g + t, t == 0, k);
        }
        commit_pair(da_full);
        g += nt;
        x += nt;
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------------ epilogue (kNWG warpgroups)
    // warpgroup wg: columns [CW wg, CW wg + CW) of every tile, the same share of A's K and of
    // dA's D; 4 warpgroups = 4 warps per SMSP to hide the per-logit MUFU / TMEM latencies
    constexpr int CW = BNT / kNWG;                        // tile columns per warpgroup
    constexpr int DQ = D / kNWG;                          // dA columns per warpgroup
    const int wg = (warp - 2) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;                          // row within this CTA's 128 rows
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool fac_fast = *p.fac_ok != 0;
    const int c0 = CW * wg;
    const uint32_t s_empty_l = mapa(smem_u32(s_empty), 0), w_full_l = mapa(smem_u32(w_full), 0);   // s: + 8 b
    const uint32_t da_empty_l = mapa(smem_u32(da_empty), 0);
    int g = 0, k = 0;
    int prev_side = 0, prev_rb = 0, prev_slot = 0;
    auto readout = [&](int side, int rb, int slot, int kk) {
      mbar_wait(da_full, kk & 1);
      tc_fence_after();
      const int row = rb * 256 + 128 * (int)rank + r;
      const Grad2Side& sd = p.side[side];
      const bool rv = row < p.Na;
      float* out = sd.part_da + ((size_t)slot * p.Na + row) * D + DQ * wg;
#pragma unroll 1
      for (int c = 0; c < DQ / 32; ++c) {
        uint32_t v[32];
        tmem_ld32_nowait(tm_da + lane_off + DQ * wg + 32 * c, v);
        tmem_ld_wait();
        if (rv) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(out + 32 * c)[i] =
                make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                            __uint_as_float(v[4 * i + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_remote(da_empty_l);
    };
    for (long x = x0; x < x1; ++k) {
      int side, rb, tb, nt;
      unit_at(x, side, rb, tb, nt);
      const Grad2Side& sd = p.side[side];
      const int row = rb * 256 + 128 * (int)rank + r;
      const bool rv = row < p.Na;
      if (k > 0) readout(prev_side, prev_rb, prev_slot, k - 1);
      const g2::RowConst<ENERGY> kc(sd, row, rv, p.invN, fac_fast);
      float wsum = 0.f;
      for (int t = 0; t < nt; ++t, ++g) {
        const int sl = g & 1;
        const int j0 = (tb + t) * BNT;
        const int nval = p.Nb - j0;
        const int sb = g & 1;
        mbar_wait(&s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        const bool tl = warp == 2 && lane == 0;
        if (tl) g2::g2_trace(p.trace, g, 4);
        uint32_t raw[CW];
#pragma unroll
        for (int h = 0; h < CW / 32; ++h)
          tmem_ld32_nowait(tm_s + 128u * (uint32_t)sb + lane_off + c0 + 32 * h,
                           *reinterpret_cast<uint32_t(*)[32]>(raw + 32 * h));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_remote(s_empty_l + 8u * (uint32_t)sb);
        if (tl) g2::g2_trace(p.trace, g, 5);
        mbar_wait(&st_full[sl], (g >> 1) & 1);
        const float* bst = sStat + sl * STAT_FLOATS;
        uint32_t pk[CW / 2];
        if (p.dbg & 1) {
#pragma unroll
          for (int i = 0; i < CW / 2; ++i) pk[i] = raw[2 * i] ^ raw[2 * i + 1];
        } else {
          g2::w_tile<ENERGY, CW, RQ>(raw, bst, c0, nval, fac_fast && nval >= BNT, fac_fast, kc, sd.lc + j0, pk, wsum);
        }
        if (tl) g2::g2_trace(p.trace, g, 6);
        if (g >= 1) mbar_wait(w_empty, (g - 1) & 1);        // dA(g - 1) (and its W store) read W
        const uint32_t wt = smem_u32(sW + (c0 >> 6) * W_CH);  // K-chunk of these columns
#pragma unroll
        for (int u = 0; u < CW / 8; ++u)
          g2::sts_u4(wt + g2::sw128_off(r, (c0 & 63) + 8 * u),
                     make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          arrive_remote(w_full_l);
          mbar_arrive(&st_empty[sl]);
          if (wst) mbar_arrive(w_loc);
        }
        if (tl) g2::g2_trace(p.trace, g, 7);
      }
      // partial slot = the piece of the row block: 0 for the piece at its first tile, else the
      // number of pair ranges that began inside the row block up to this one (<= 2: one side only
      // gives a pair >= half a row-block pair of tiles)
      int slot = 0;
      if (tb != 0) {
        const long first = x - (long)tb;
        int pf = cid;
        while (pf > 0 && g2::range_start(pf, X, ncl) > first) --pf;
        slot = cid - pf;
      }
      if ((ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) && rv)
        sd.part_rs[((size_t)(kNWG * slot + wg)) * p.Na + row] = wsum;
      prev_side = side; prev_rb = rb; prev_slot = slot;
      x += nt;
    }
    if (k > 0) readout(prev_side, prev_rb, prev_slot, k - 1);
  }
  tc_fence_before();
  cluster_sync();                          // the peer's MMAs / arrivals are done before TMEM goes
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ------------------------------------------------------------------------------- host side
int tc_grad2_grid(int Na, int num_sms) {
  const int RB = (Na + 127) / 128;
  // at most 2 pieces per row block: every CTA's range spans >= one row block's tiles
  return std::max(1, std::min(num_sms, 2 * RB));
}

// slot-1 flags: row block rb of side s is cut by a CTA boundary (its second piece -> slot 1)
void tc_grad2_split_flags(int Na, int Nb, int grid, unsigned char* flags /*[2][RB]*/) {
  const long RB = (Na + 127) / 128, TPB = (Nb + g2::BNT - 1) / g2::BNT, X = 2 * RB * TPB;
  for (long r = 0; r < 2 * RB; ++r) {
    const long first = r * TPB, last = first + TPB - 1;
    bool cut = false;
    for (long c = 1; c < grid; ++c) {
      const long st = g2::range_start(c, X, grid);
      if (st > first && st <= last) { cut = true; break; }
    }
    flags[r] = cut ? 1 : 0;
  }
}

template <int ENERGY>
static cudaError_t launch_g2(const CUtensorMap& b0, const CUtensorMap& b1, const Grad2Args& p, int grid,
                             cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_grad2_kernel<ENERGY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)g2::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(tc_grad2_kernel<ENERGY>, dim3(grid), dim3(352), g2::SMEM, st, b0, b1, p);
}

int tc_grad2p_warpgroups() { return g2p::kNWG; }

// ---- CTA pairs: a pair owns 256-row row-block PAIRS; grid = 2 x pairs
int tc_grad2p_grid(int Na, int num_sms) {
  const int RBP = (Na + 255) / 256;
  return 2 * std::max(1, std::min(num_sms / 2, 2 * RBP));
}
// slot-1 flags per 128-row block: a row-block pair cut by a pair boundary flags both its blocks
int tc_grad2p_split_flags(int Na, int Nb, int grid, unsigned char* flags /*[2][RB]*/, int nsides) {
  const long RB = (Na + 127) / 128, RBP = (Na + 255) / 256, TPB = (Nb + g2::BNT - 1) / g2::BNT;
  const long X = (nsides == 1 ? 1 : 2) * RBP * TPB, P = grid / 2;
  int pieces = 1;
  for (long side = 0; side < 2; ++side)
    for (long rb = 0; rb < RB; ++rb) {
      const long rp = side * RBP + rb / 2, first = rp * TPB, last = first + TPB - 1;
      int cuts = 0;                                       // pair ranges beginning inside the row block
      for (long c = 1; c < P; ++c) {
        const long st = g2::range_start(c, X, P);
        if (st > first && st <= last) ++cuts;
      }
      flags[side * RB + rb] = (unsigned char)cuts;
      if (first < X) pieces = std::max(pieces, 1 + cuts);
    }
  return pieces;
}

template <int ENERGY, int RQ>
static cudaError_t launch_g2p(const CUtensorMap& d0, const CUtensorMap& d1, const CUtensorMap& s0,
                              const CUtensorMap& s1, const CUtensorMap& a0, const CUtensorMap& a1,
                              const CUtensorMap& w, const Grad2Args& p, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_grad2p_kernel<ENERGY, RQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)g2p::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(tc_grad2p_kernel<ENERGY, RQ>, dim3(grid), dim3(128 + 128 * g2p::kNWG), g2p::SMEM, st, d0, d1, s0,
                    s1, a0, a1, w, p);
}

cudaError_t tc_grad2p(int energy, const CUtensorMap& mD0, const CUtensorMap& mD1, const CUtensorMap& mS0,
                      const CUtensorMap& mS1, const CUtensorMap& mA0, const CUtensorMap& mA1, const Grad2Args& p0,
                      int grid, cudaStream_t st, const CUtensorMap* mW) {
  Grad2Args p = p0;
  if (const char* d = std::getenv("CRL_G2P_DBG")) p.dbg = std::atoi(d);   // measurement ablations
  static const CUtensorMap kNoMap{};
  if (p.w_store && (mW == nullptr || p.nsides != 1)) return cudaErrorInvalidValue;
  const CUtensorMap& w = mW != nullptr ? *mW : kNoMap;
  p.RB = (p.Na + 255) / 256;                              // row-block PAIRS
  p.TPB = (p.Nb + g2p::BNT - 1) / g2p::BNT;
  if (energy == CRL_ENERGY_L2) {
    // L2: of every 4 logit pairs, RQ take rsqrt on the FMA pipe instead of the MUFU
    const int rq = std::getenv("CRL_G2_RSQ") ? std::atoi(std::getenv("CRL_G2_RSQ")) : g2::kG2RsqPairs;
    switch (rq) {
      case 1: return launch_g2p<CRL_ENERGY_L2, 1>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
      case 2: return launch_g2p<CRL_ENERGY_L2, 2>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
      case 3: return launch_g2p<CRL_ENERGY_L2, 3>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
      case 4: return launch_g2p<CRL_ENERGY_L2, 4>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
      default: return launch_g2p<CRL_ENERGY_L2, 0>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
    }
  }
  if (energy == CRL_ENERGY_L2SQ) return launch_g2p<CRL_ENERGY_L2SQ, 0>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
  if (energy == CRL_ENERGY_COS) return launch_g2p<CRL_ENERGY_COS, 0>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
  return launch_g2p<CRL_ENERGY_DOT, 0>(mD0, mD1, mS0, mS1, mA0, mA1, w, p, grid, st);
}

cudaError_t tc_grad2(int energy, const CUtensorMap& mB0, const CUtensorMap& mB1, const Grad2Args& p0, int grid,
                     cudaStream_t st) {
  Grad2Args p = p0;
  p.RB = (p.Na + 127) / 128;
  p.TPB = (p.Nb + g2::BNT - 1) / g2::BNT;
  if (energy == CRL_ENERGY_L2) return launch_g2<CRL_ENERGY_L2>(mB0, mB1, p, grid, st);
  if (energy == CRL_ENERGY_L2SQ) return launch_g2<CRL_ENERGY_L2SQ>(mB0, mB1, p, grid, st);
  if (energy == CRL_ENERGY_COS) return launch_g2<CRL_ENERGY_COS>(mB0, mB1, p, grid, st);
  return launch_g2<CRL_ENERGY_DOT>(mB0, mB1, p, grid, st);
}

}  // namespace tc
}  // namespace crl
