// tc_pgemm.cu — persistent CTA-pair (tcgen05 cta_group::2) GEMM for the wide encoder layers of
// the BF16 path (SURVEY §8(a) A2 forward and A5 dX at width 1024: configs[4], §5.4 P:387-465,
// Table 2).
//
//   forward  Z[M][N] = X[M][K] . W[K][N] + b     A = X  K-major, B = W MN-major (as stored)
//            hidden: Z (bf16) and act(Z) (bf16);  output layer: Y fp32 + Y bf16 + row statistic
//   dX       dZp[M][N] = (dZ[M][K] . W[N][K]^T) * act'(Zp)   A = dZ K-major, B = W K-major
//
// Anatomy.  A cluster of 2 CTAs (a TPC pair) owns one 256 x 256 output tile at a time and walks
// the tile list persistently (tile t = cluster id + k * #clusters, N fastest so the pairs that
// run together share their A rows in L2).  The MMA is tcgen05.mma.cta_group::2 (M = 256,
// N = 256, K = 16): CTA r of the pair stages rows [128 r, 128 r + 128) of A and columns
// [128 r, 128 r + 128) of B, so each SM reads half the operand bytes of a 1-CTA 128 x 256 tile
// from its kSmem and the L2 -> kSmem traffic per tile is halved; each CTA's TMEM receives its
// 128 rows x 256 columns of the accumulator.
//   warp 0 (lane 0, both CTAs)  TMA producer: 5-stage ring of 64-wide K blocks (32 KB / stage /
//                               CTA); completion bytes of BOTH CTAs land on the leader's full
//                               barrier (cta_group::2 TMA)
//   warp 1 (lane 0, leader)     MMA issuer; stage release and accumulator-ready commits are
//                               multicast to both CTAs
//   warps 2..5 (both CTAs)      epilogue: TMEM lane quarter q = warp & 3 (32 rows), 64-column
//                               chunks: tcgen05.ld -> bias / activation / activation' -> bf16
//                               (fp32) SW128 staging -> TMA tensor stores (DX: the Z_prev chunk
//                               arrives by TMA into the same staging buffer first)
//   TMEM: two 256-column fp32 accumulators (512 columns): tile t's epilogue overlaps tile
//   t + 1's mainloop; the leader's MMA waits on an "accumulator empty" barrier that all 8
//   epilogue warps of the pair arrive on.
// Measured bound (scratch/pgemm_test.cu ablations, 16384 x 1024 x 1024 hidden layer): 37 us
// whole, 22.7 us without the epilogue (the MMA floor at 128 B/clk of SMEM operand traffic:
// TMA writes + MMA reads of 2 x 16 KB per 512-cycle K block), 25.5 us epilogue alone.  Tried
// and not kept: 3-6 stages x 1-8 staging buffers (all within +-3 %), register -> global stores
// of Z / act(Z) (16 B stores 52 us, 32 B STG.256 38 us).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_pgemm.h"
#include "tc_pair.cuh"

namespace crl {
namespace tc {
namespace pg {
using namespace pair;

constexpr int kBK = 64, kStages = 5, kTN = 256;      // K block, ring depth, tile N (= tile M / 1)
constexpr uint32_t kAHalf = 128 * kBK * 2;          // 16 KB: this CTA's 128 rows of A
constexpr uint32_t kBHalf = 128 * kBK * 2;          // 16 KB: this CTA's 128 columns of B
constexpr uint32_t kStage = kAHalf + kBHalf;
constexpr uint32_t kStgBuf = 32 * 128;             // 4 KB: 32 rows x 128 B (SW128) staging
// epilogue warps EW: 4 (one per TMEM lane quarter, 4 staging buffers each) or 8 (two per
// quarter, every other 64-column chunk each, 2 buffers): the same 64 KB of staging.  Measured on
// B200 (scratch/pgemm_test.cu, 16384 x 1024 x 1024): 34.3 us with 4, 35.0 with 8 -- an SMEM-bound
// mainloop leaves the epilogue no bandwidth to gain; the short-K layers (K <= 256: the first
// layer, the output layer's dX) are epilogue-bound and take 8
template <int EW>
struct Epi {
  static constexpr int kEpiW = EW;
  static constexpr int kNStg = EW == 8 ? 2 : 4;     // staging buffers per epilogue warp
};
constexpr size_t kSmem = 1024 + kStages * kStage + 16 * kStgBuf + 256;

// number of 64-column chunks c = h, h + nh, ... below nch (a warp's chunks in one tile)
__host__ __device__ __forceinline__ int ci_count(int nch, int h, int nh) { return nch > h ? (nch - 1 - h) / nh + 1 : 0; }
__device__ __forceinline__ void tma_load_2d_local(uint32_t dst, const CUtensorMap* map, uint64_t* mbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(mbar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void expect_tx_remote(uint32_t mbar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(mbar_cluster), "r"(bytes) : "memory");
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

}  // namespace pg

template <int EPI, int ACT, int EW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * EW, 1)
    tc_pgemm_kernel(const __grid_constant__ PgemmJob J) {
  using namespace pg;
  constexpr int kEpiW = Epi<EW>::kEpiW, kNStg = Epi<EW>::kNStg;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = smem;
  uint8_t* sStg = sStage + kStages * kStage;                         // [kEpiW warps][kNStg][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + kEpiW * kNStg * kStgBuf);
  uint64_t* full = bars;                  // [kStages]  leader: both CTAs' TMA bytes
  uint64_t* empty = full + kStages;        // [kStages]  both: MMA commit (multicast)
  uint64_t* tfull = empty + kStages;       // [2]       both: accumulator ready (multicast)
  uint64_t* tempty = tfull + 2;           // [2]       leader: 8 epilogue warps of the pair
  uint64_t* zbar = tempty + 2;            // [kEpiW][kNStg] DX: Z_prev chunk landed (per warp)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zbar + kEpiW * kNStg);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int n_tiles = J.total;
  // tile t of the job: problem pi, local tile tt; that problem's maps / arguments / shape
#define PG_TILE(t)                                                    \
  const int pi = (J.np > 1 && (t) >= J.nt0) ? 1 : 0;                  \
  const int tt = (t) - (pi ? J.nt0 : 0);                              \
  const PgemmMaps& maps = J.maps[pi];                                 \
  const PgemmArgs& p = J.args[pi];                                    \
  const int tiles_n = (p.N + kTN - 1) / kTN;                          \
  const int nkb = (p.K + kBK - 1) / kBK;                              \
  (void)maps; (void)nkb; (void)tiles_n;
  const PgemmArgs& p0 = J.args[0];

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < J.np; ++i) { tma_prefetch_desc(&J.maps[i].a); tma_prefetch_desc(&J.maps[i].b); }
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * kEpiW); }
    for (int i = 0; i < kEpiW * kNStg; ++i) mbar_init(&zbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();                          // both CTAs' barriers and TMEM exist
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();
  if (p0.trace && threadIdx.x == 0 && rank == 0) p0.trace[512 + 2 * cid] = (long long)globaltimer();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      const uint32_t full_leader = mapa(smem_u32(full), 0);
      int g = 0;
      for (int t = cid; t < n_tiles; t += ncl) {
        PG_TILE(t)
        const int m0 = (tt / tiles_n) * 256 + 128 * (int)rank;
        const int n0 = (tt % tiles_n) * kTN + 128 * (int)rank;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
          const uint32_t fb = full_leader + 8u * (uint32_t)s;
          if (p.dbg & 4) {                                 // ablation: no operand traffic
            if (rank == 0) mbar_arrive(&full[s]);
            continue;
          }
          if (rank == 0) mbar_expect_tx(&full[s], 2 * kStage);
          const uint32_t a_dst = smem_u32(sStage + s * kStage);
          const uint32_t b_dst = a_dst + kAHalf;
          const int k = kb * kBK;
          tma_load_2d_pair(a_dst, &maps.a, fb, k, m0);                       // A {K, M} box {64, 128}
          if (EPI == PG_DX) {
            tma_load_2d_pair(b_dst, &maps.b, fb, k, n0);                     // W {K=out, N=in} box {64, 128}
          } else {
            tma_load_2d_pair(b_dst, &maps.b, fb, n0, k);                     // W {N, K} box {64, 64} x 2
            tma_load_2d_pair(b_dst + kBK * 128, &maps.b, fb, n0 + 64, k);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ------------------------------------------------------------------ MMA issuer (leader)
      const uint32_t idesc = idesc_bf16_f32(256, kTN, false, EPI != PG_DX);
      int g = 0, it = 0;
      for (int t = cid; t < n_tiles; t += ncl, ++it) {
        PG_TILE(t)
        const int b = it & 1;
        mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + 256u * (uint32_t)b;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait(&full[s], (g / kStages) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sStage + s * kStage);
          const uint32_t b_base = a_base + kAHalf;
          if (!(p.dbg & 2))
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            const uint64_t ad = smem_desc_sw128(a_base + ks * 32, 16, 1024);
            const uint64_t bd = EPI == PG_DX ? smem_desc_sw128(b_base + ks * 32, 16, 1024)
                                             : smem_desc_sw128(b_base + ks * 2048, kBK * 128, 1024);
            mma_pair(d, ad, bd, idesc, (kb | ks) != 0);
          }
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[b]);
        if (p0.trace && cid == 0 && it < 8) p0.trace[256 + it] = clock64();
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;                               // TMEM lane quarter = 32 rows
    const int ew = warp - 2;                              // staging owner index
    constexpr int nh = kEpiW / 4;                         // warps per lane quarter
    const int h = ew / 4;                                 // this warp's chunks: c = h, h + nh, ...
    const uint32_t stg0 = smem_u32(sStg + (size_t)ew * kNStg * kStgBuf);
    // output layer: the h = 0 warps take every chunk with 3 buffers each, borrowing the staging
    // of their h = 1 partner (idle there) when kNStg = 2
    const uint32_t stgX = smem_u32(sStg + (size_t)((ew + 4) % kEpiW) * kNStg * kStgBuf);
    auto obuf = [&](int i) -> uint32_t { return i < kNStg ? stg0 + i * kStgBuf : stgX + (i - kNStg) * kStgBuf; };
    const int c_first = EPI == PG_FWD_OUT ? 0 : h, c_step = EPI == PG_FWD_OUT ? 1 : nh;
    const bool active = EPI != PG_FWD_OUT || h == 0;
    uint64_t* zb = zbar + ew * kNStg;
    const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
    const uint32_t row_sw = (uint32_t)((lane >> 3) * 1024 + (lane & 7) * 128);   // SW128 row base
    int it = 0;
    uint32_t zphase = 0;                                   // DX: parity bits of zb[] (one per buffer)
    for (int t = cid; t < n_tiles; t += ncl, ++it) {
      PG_TILE(t)
      const int b = it & 1;
      const int mrow0 = (tt / tiles_n) * 256 + 128 * (int)rank + 32 * q;   // first row of this warp
      const int ncol0 = (tt % tiles_n) * kTN;
      const int nch = min(kTN, p.N - ncol0) / 64;         // 64-column chunks (N % 64 == 0)
      if (EPI == PG_DX && lane == 0) {
        // Z_prev chunks of this warp for this tile: issued before the accumulator is ready
        // (latency hidden behind the mainloop); buffer i holds the warp's i-th chunk
        bulk_wait_read<0>();                              // staging reads of the last tile done
        for (int c = h, i = 0; c < nch; c += nh, ++i) {
          mbar_expect_tx(&zb[i], kStgBuf);
          tma_load_2d_local(stg0 + i * kStgBuf, &maps.zin, &zb[i], ncol0 + 64 * c, mrow0);
        }
      }
      if (EPI != PG_DX && lane == 0) bulk_wait_read<0>();  // staging of the previous tile read
      __syncwarp();
      mbar_wait(&tfull[b], (it >> 1) & 1);
      tc_fence_after();
      const bool trc = p.trace && cid == 0 && rank == 0 && ew == 0 && lane == 0 && it < 8;
      if (trc) p.trace[264 + it] = clock64();
      float ysq = 0.f;
      // a warp without chunks in this tile (or the idle half at the output layer) releases the
      // accumulator right away: every epilogue warp arrives once per tile
      const int c_last = !active || c_first >= nch ? -1 : c_first + ((nch - 1 - c_first) / c_step) * c_step;
      if ((EPI != PG_DX && (p.dbg & 1)) || c_last < 0) {  // (dbg & 1: ablation, accumulator dropped)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_remote(tempty_leader + 8u * (uint32_t)b);
        continue;
      }
      // software pipeline over the warp's 64-column chunks: chunk c + c_step's TMEM load (and
      // bias load) is in flight while chunk c is processed
      const uint32_t tbase = tmem + 256u * (uint32_t)b + ((uint32_t)(q * 32) << 16);
      uint32_t v[64];
      float4 bb[16];
      auto issue = [&](int c) {
        tmem_ld32_nowait(tbase + 64u * (uint32_t)c, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32_nowait(tbase + 64u * (uint32_t)c + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        if (EPI != PG_DX) {                              // bias (broadcast: every lane the same column)
#pragma unroll
          for (int i4 = 0; i4 < 16; ++i4) bb[i4] = __ldg(reinterpret_cast<const float4*>(p.bias + ncol0 + 64 * c) + i4);
        }
      };
      // 4 epilogue warps: chunk c + c_step's loads in flight while chunk c is processed; 8 warps
      // (two per lane quarter hide each other's latency) load chunk by chunk (register budget)
      constexpr bool kPipe = EW == 4;
      if (kPipe) issue(c_first);
      for (int c = c_first, ci = 0; c < nch; c += c_step, ++ci) {
        if (!kPipe) issue(c);
        tmem_ld_wait();
        if (trc && c < 4) p.trace[(it * 4 + c) * 4 + 0] = clock64();
        f32x2 f2[32];                                     // the chunk's 64 values as packed pairs
#pragma unroll
        for (int i = 0; i < 32; ++i) f2[i] = f2_pack(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        if (EPI != PG_DX) {
#pragma unroll
          for (int i4 = 0; i4 < 16; ++i4) {
            f2[2 * i4] = f2_add(f2[2 * i4], f2_pack(bb[i4].x, bb[i4].y));
            f2[2 * i4 + 1] = f2_add(f2[2 * i4 + 1], f2_pack(bb[i4].z, bb[i4].w));
          }
        }
        if (c == c_last) {                                // accumulator b free for tile it + 2
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_remote(tempty_leader + 8u * (uint32_t)b);
        } else {
          if (kPipe) issue(c + c_step);
        }
        const int n = ncol0 + 64 * c;
        if (EPI == PG_DX) {
          // dZ_prev = acc * act'(Z_prev); Z_prev from the staging buffer, result written back in place
          mbar_wait(&zb[ci], (zphase >> ci) & 1);
          const uint32_t buf = stg0 + ci * kStgBuf + row_sw;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t addr = buf + (uint32_t)(((j ^ (lane & 7))) << 4);
            const uint4 zz = lds128(addr);
            const uint32_t w[4] = {zz.x, zz.y, zz.z, zz.w};
            uint32_t o[4];
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
              const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[hh]));
              f32x2 a = f2[4 * j + hh];
              if (ACT == CRL_ACT_SILU) {
                // SiLU'(z) = s (1 + z (1 - s)) = 1/2 + (h (1 - t^2) + t) / 2,  h = z / 2, t = tanh h
                const f32x2 hz = f2_mul(f2_pack(z.x, z.y), f2_pack(0.5f, 0.5f));
                float h0, h1;
                f2_unpack(hz, h0, h1);
                const f32x2 t = f2_pack(pg::tanh_approx(h0), pg::tanh_approx(h1));
                const f32x2 om = f2_fma(f2_mul(t, f2_pack(-1.f, -1.f)), t, f2_pack(1.f, 1.f));
                const f32x2 g = f2_fma(f2_pack(0.5f, 0.5f), f2_fma(hz, om, t), f2_pack(0.5f, 0.5f));
                a = f2_mul(a, g);
              } else {
                float a0, a1;
                f2_unpack(a, a0, a1);
                a = f2_pack(z.x > 0.f ? a0 : 0.f, z.y > 0.f ? a1 : 0.f);
              }
              float a0, a1;
              f2_unpack(a, a0, a1);
              o[hh] = pack_bf16x2(a0, a1);
            }
            sts128(addr, make_uint4(o[0], o[1], o[2], o[3]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&maps.out0, stg0 + ci * kStgBuf, n, mrow0);
            bulk_commit();
          }
        } else if (EPI == PG_FWD_HIDDEN) {
          // buffers: Z chunk, act(Z) chunk (2 x 4 KB) at (2c) % kNStg and (2c+1) % kNStg; the warp's
          // chunk ci uses those of chunk ci - kNStg / 2, which must have been read by their stores
          if (lane == 0 && ci >= kNStg / 2) bulk_wait_read<kNStg / 2 - 1>();
          __syncwarp();
          if (trc && c < 4) p.trace[(it * 4 + c) * 4 + 1] = clock64();
          const uint32_t bz = stg0 + ((2 * ci) % kNStg) * kStgBuf + row_sw;
          const uint32_t bx = stg0 + ((2 * ci + 1) % kNStg) * kStgBuf + row_sw;
          const bool lin = p.lin != 0, noact = (p.dbg & 16) != 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (uint32_t)(((j ^ (lane & 7))) << 4);
            uint32_t oz[4], ox[4];
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
              const f32x2 z = f2[4 * j + hh];
              float z0, z1;
              f2_unpack(z, z0, z1);
              oz[hh] = pack_bf16x2(z0, z1);
              if (ACT == CRL_ACT_SILU) {                  // SiLU(z) = h + h tanh(h), h = z / 2
                const f32x2 hz = f2_mul(z, f2_pack(0.5f, 0.5f));
                float h0, h1;
                f2_unpack(hz, h0, h1);
                float x0, x1;
                f2_unpack(f2_fma(hz, f2_pack(pg::tanh_approx(h0), pg::tanh_approx(h1)), hz), x0, x1);
                ox[hh] = pack_bf16x2(x0, x1);
              } else {
                ox[hh] = pack_bf16x2(fmaxf(z0, 0.f), fmaxf(z1, 0.f));
              }
              if (noact) ox[hh] = oz[hh];                  // ablation: no activation math
            }
            sts128(bz + off, make_uint4(oz[0], oz[1], oz[2], oz[3]));
            if (!lin) sts128(bx + off, make_uint4(ox[0], ox[1], ox[2], ox[3]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (trc && c < 4) p.trace[(it * 4 + c) * 4 + 2] = clock64();
          if (lane == 0 && !(p.dbg & 8)) {               // (dbg & 8: ablation, no output stores)
            tma_store_2d(&maps.out0, bz - row_sw, n, mrow0);
            if (!lin) tma_store_2d(&maps.out1, bx - row_sw, n, mrow0);
            bulk_commit();
          }
        } else {                                          // PG_FWD_OUT
          if (lane == 0 && c >= 1) bulk_wait_read<0>();  // chunk c - 1's staging is read
          __syncwarp();
          const uint32_t by = obuf(0) + row_sw;                      // bf16 Y
          const uint32_t bf0 = obuf(1) + row_sw;                     // fp32 Y columns 0..31
          const uint32_t bf1 = obuf(2) + row_sw;                     // fp32 Y columns 32..63
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (uint32_t)(((j ^ (lane & 7))) << 4);
            float y[8];
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) f2_unpack(f2[4 * j + hh], y[2 * hh], y[2 * hh + 1]);
            const uint4 hb = make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]),
                                        pack_bf16x2(y[6], y[7]));
            sts128(by + off, hb);
            // the logits stage's row statistic is taken on the bf16-rounded Y it will read
            const uint32_t w[4] = {hb.x, hb.y, hb.z, hb.w};
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
              const float2 yb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[hh]));
              ysq = fmaf(yb.x, yb.x, fmaf(yb.y, yb.y, ysq));
            }
            // fp32: 8 floats = 2 x 16 B chunks of the 32-column half j / 4
            const uint32_t bfh = (j < 4) ? bf0 : bf1;
            const int c16 = 2 * (j & 3);
            sts128(bfh + (uint32_t)(((c16 ^ (lane & 7))) << 4),
                   make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]), __float_as_uint(y[3])));
            sts128(bfh + (uint32_t)((((c16 + 1) ^ (lane & 7))) << 4),
                   make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]), __float_as_uint(y[6]), __float_as_uint(y[7])));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&maps.out1, by - row_sw, n, mrow0);
            tma_store_2d(&maps.out0, bf0 - row_sw, n, mrow0);
            tma_store_2d(&maps.out0, bf1 - row_sw, n + 32, mrow0);
            bulk_commit();
          }
        }
      }
      if (EPI == PG_DX) zphase ^= (1u << (ci_count(nch, h, nh))) - 1u;
      if (EPI == PG_FWD_OUT && p.stat != nullptr) {
        const int row = mrow0 + lane;
        if (row < p.M)
          p.stat[row] = (p.stat_energy == CRL_ENERGY_L2 || p.stat_energy == CRL_ENERGY_L2SQ) ? ysq
                        : (p.stat_energy == CRL_ENERGY_COS ? 1.f / fmaxf(sqrtf(ysq), kEpsCos) : 0.f);
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync();                          // the peer's MMAs / arrivals are done before TMEM goes
  if (p0.trace && threadIdx.x == 0 && rank == 0) p0.trace[512 + 2 * cid + 1] = (long long)globaltimer();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// -------------------------------------------------------------------------------- host side
// M: rows (any, >= 256 so a pair has work), N: a multiple of 64 (whole staging chunks), >= 256
// (the 256-wide tile; narrower layers keep tc_gemm), K: any (TMA zero-fills the last K block)
bool tc_pgemm_supported(int M, int N, int K) {
  return M >= 256 && N >= 256 && N % 64 == 0 && K >= 1 && !std::getenv("CRL_NO_PGEMM");
}

template <int EPI, int ACT, int EW>
static cudaError_t launch_pg(const PgemmJob& J, int num_sms, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_pgemm_kernel<EPI, ACT, EW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pg::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int clusters = std::max(1, std::min(J.total, num_sms / 2));
  return launch_pdl(tc_pgemm_kernel<EPI, ACT, EW>, dim3(2 * clusters), dim3(64 + 32 * EW), pg::kSmem, st, J);
}
template <int EPI, int ACT>
static cudaError_t launch_pg_ew(const PgemmJob& J, int num_sms, cudaStream_t st) {
  // short K (<= 256): the epilogue is the bound, twice the epilogue warps
  int kmax = J.args[0].K;
  if (J.np > 1) kmax = std::max(kmax, J.args[1].K);
  const char* e = std::getenv("CRL_PG_EPIW");
  const int ew = e ? std::atoi(e) : (kmax <= 256 ? 8 : 4);
  if (ew == 8) return launch_pg<EPI, ACT, 8>(J, num_sms, st);
  return launch_pg<EPI, ACT, 4>(J, num_sms, st);
}
template <int EPI>
static cudaError_t launch_pg_act(const PgemmJob& J, int num_sms, cudaStream_t st) {
  if (EPI == PG_FWD_OUT || J.args[0].act == CRL_ACT_SILU) return launch_pg_ew<EPI, CRL_ACT_SILU>(J, num_sms, st);
  return launch_pg_ew<EPI, CRL_ACT_RELU>(J, num_sms, st);
}
static int pg_tiles(const PgemmArgs& p) { return ((p.M + 255) / 256) * ((p.N + pg::kTN - 1) / pg::kTN); }

static cudaError_t pg_run(int epi, const PgemmJob& J, int num_sms, cudaStream_t st) {
  switch (epi) {
    case PG_FWD_HIDDEN: return launch_pg_act<PG_FWD_HIDDEN>(J, num_sms, st);
    case PG_FWD_OUT: return launch_pg_act<PG_FWD_OUT>(J, num_sms, st);
    case PG_DX: return launch_pg_act<PG_DX>(J, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t tc_pgemm(int epi, const PgemmMaps& maps, const PgemmArgs& p, int num_sms, cudaStream_t st) {
  PgemmJob J{};
  J.maps[0] = maps;
  J.args[0] = p;
  J.np = 1;
  J.nt0 = J.total = pg_tiles(p);
  return pg_run(epi, J, num_sms, st);
}

cudaError_t tc_pgemm2(int epi, const PgemmMaps& maps0, const PgemmArgs& p0, const PgemmMaps& maps1,
                      const PgemmArgs& p1, int num_sms, cudaStream_t st) {
  if (p0.act != p1.act) return cudaErrorInvalidValue;
  PgemmJob J{};
  J.maps[0] = maps0;
  J.maps[1] = maps1;
  J.args[0] = p0;
  J.args[1] = p1;
  J.np = 2;
  J.nt0 = pg_tiles(p0);
  J.total = J.nt0 + pg_tiles(p1);
  return pg_run(epi, J, num_sms, st);
}

}  // namespace tc
}  // namespace crl
