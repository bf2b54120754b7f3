// tc_pdw.cu — every weight and bias gradient of the WIDE encoders on CTA pairs (A5, BF16 path,
// configs[4]: 4 x 1024 hidden layers, §5.4).
//
// Paper: backward of the encoders of §3.1 P:193-195 (Alg. 1 P:1051 "gradient"):
//   dW_l = X_l^T dZ_l  (M = in, N = out, K = batch)      db_l = 1^T dZ_l  (column sums)
//
// The grouped single-CTA kernel (tc_dwg.cu) runs 128 x 256 tiles whose operands cost 96 KB of
// SMEM traffic per 512-cycle K block (188 B/clk against the 128 B/clk the SM delivers): it is
// bound at ~2/3 of the tensor rate.  Here a CLUSTER of 2 CTAs owns a 256 x 256 tile of dW
// (tcgen05.mma.cta_group::2, M = 256, N = 256, K = 16): CTA r stages in-columns
// [128 r, 128 r + 128) of X_l and out-columns [128 r, 128 r + 128) of dZ_l (both MN-major, as
// stored: no transposed copies), 64 KB of SMEM traffic per K block per SM = 128 B/clk, the MMA
// rate.  The pairs walk a static list of (problem, K slice, M tile, N tile) work items; each
// item accumulates its K slice in one of two 256-column TMEM accumulators, so item i's
// epilogue (fp32 -> SW128 staging -> 3-D TMA stores into the slice's partial buffer, summed by
// Adam: deterministic) overlaps item i + 1's mainloop.
//   warp 0 (lane 0, both CTAs)  TMA producer, 5-stage ring (32 KB / stage / CTA)
//   warp 1 (lane 0, leader)     MMA issuer; stage-consumed commits multicast to both CTAs
//   warps 2..5 (both CTAs)      epilogue (TMEM lane quarter = 32 rows of dW)
//   warps 6.. (both CTAs)       bias gradient: on items of M tile 0, the column sums of the dZ
//                               stage this CTA staged (its 128 NH out-columns), read from SMEM
//                               after the MMA consumed it (64 / kBiasW of the K block's rows each);
//                               the stage is refilled only after they arrived
// db_l is thus a by-product of dW_l's operand stream: no ones-MMA, no second pass over dZ_l.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_pair.cuh"
#include "tc_pdw.h"

namespace crl {
namespace tc {

bool make_map_bf16(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
bool make_map_f32_3d(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);

namespace pdw {
using namespace pair;

constexpr int kBK = 64;
constexpr uint32_t kHalf = 128 * kBK * 2;            // 16 KB: 128 MN-columns x 64 K rows
constexpr uint32_t kStgBuf = 32 * 128;               // 4 KB: 32 rows x 32 fp32 (SW128)
// NH 256-column halves per work item (NH = 2: 256 x 512 dW tiles, both TMEM accumulators, 25 %
// less operand traffic per flop; NH = 1: 256 x 256 tiles, double-buffered accumulators)
template <int NH>
struct Cfg {
  static constexpr int kStages = NH == 2 ? 4 : 6;
  static constexpr uint32_t kStage = kHalf * (1 + NH);           // A half + NH B halves
  static constexpr int kNStg = 2;                                // staging buffers per epilogue warp
  static constexpr int kTN = 256 * NH;                           // item width
  static constexpr int kNbuf = 2 / NH;                           // accumulator buffers
  static constexpr int kBiasW = NH == 2 ? 2 : 4;                 // bias-gradient warps (64 / kBiasW K rows each)
  static constexpr int kThreads = 192 + 32 * kBiasW;
  static constexpr size_t kSmem = kStages * kStage + 4 * kNStg * kStgBuf + kBiasW * 128 * NH * 4 + 256;
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

struct Item {
  int p, slice, tm, tn;
};
__device__ __forceinline__ Item decode(const PdwParams& P, int it) {
  Item r{};
  int p = 0;
  while (p + 1 < P.n && it >= P.prob[p].tiles) { it -= P.prob[p].tiles; ++p; }
  const PdwProblem& pr = P.prob[p];
  const int per = pr.tiles / P.splits;                // tiles of one slice
  r.p = p;
  r.slice = it / per;
  const int rem = it - r.slice * per;
  r.tm = rem / pr.tiles_n;
  r.tn = rem - r.tm * pr.tiles_n;
  return r;
}

}  // namespace pdw

template <int NH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    tc_pdw_kernel(const __grid_constant__ PdwParams P) {
  using namespace pdw;
  using C = Cfg<NH>;
  constexpr int kStages = C::kStages, kNStg = C::kNStg, kTN = C::kTN, kNbuf = C::kNbuf, kBiasW = C::kBiasW;
  constexpr uint32_t kStage = C::kStage;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sStage = smem_raw;
  uint8_t* sStg = sStage + kStages * kStage;                        // [4 warps][kNStg][4 KB]
  float* sDb = reinterpret_cast<float*>(sStg + 4 * kNStg * kStgBuf);  // [kBiasW][128 NH] bias partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDb + kBiasW * 128 * NH);
  uint64_t* full = bars;                  // [kStages]  leader: both CTAs' TMA bytes
  uint64_t* empty = full + kStages;        // [kStages]  both: MMA commit + the bias warps
  uint64_t* used = empty + kStages;        // [kStages]  both: MMA commit (the bias warps may read)
  uint64_t* tfull = used + kStages;        // [kNbuf]   both: accumulator(s) ready
  uint64_t* tempty = tfull + 2;           // [kNbuf]   leader: the 8 epilogue warps of the pair
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int nkb_all = (P.K + kBK - 1) / kBK;
  auto kb_range = [&](int slice, int& kb0, int& kb1) {
    kb0 = slice * P.kb_per_split;
    kb1 = min(nkb_all, kb0 + P.kb_per_split);
  };

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();   // SW128 operand tiles need 1 KB alignment
    for (int p = 0; p < P.n; ++p) { tma_prefetch_desc(&P.prob[p].a); tma_prefetch_desc(&P.prob[p].b); }
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1 + kBiasW); mbar_init(&used[s], 1); }
    for (int i = 0; i < kNbuf; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer (both CTAs)
      const uint32_t full_leader = mapa(smem_u32(full), 0);
      int g = 0;
      for (int it = cid; it < P.total; it += ncl) {
        const Item w = decode(P, it);
        const PdwProblem& pr = P.prob[w.p];
        const int m0 = w.tm * 256 + 128 * (int)rank;
        // halves with columns (an N = 256 layer in a 512-wide item: its second half is skipped)
        const int nhi = (NH == 2 && w.tn * kTN + 256 >= pr.N) ? 1 : NH;
        int kb0, kb1;
        kb_range(w.slice, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
          if (P.dbg & 4) { if (rank == 0) mbar_arrive(&full[s]); continue; }
          if (rank == 0) mbar_expect_tx(&full[s], 2 * kHalf * (1 + nhi));
          const uint32_t fb = full_leader + 8u * (uint32_t)s;
          const uint32_t a_dst = smem_u32(sStage + s * kStage);
          const int k = kb * kBK;
          tma_load_2d_pair(a_dst, &pr.a, fb, m0, k);                 // X {in, K} box {64, 64} x 2
          tma_load_2d_pair(a_dst + kBK * 128, &pr.a, fb, m0 + 64, k);
#pragma unroll
          for (int h = 0; h < NH; ++h) {                             // dZ {out, K} box {64, 64} x 2 per half
            if (h >= nhi) break;
            const int n0 = w.tn * kTN + 256 * h + 128 * (int)rank;
            const uint32_t b_dst = a_dst + kHalf * (1 + h);
            tma_load_2d_pair(b_dst, &pr.b, fb, n0, k);
            tma_load_2d_pair(b_dst + kBK * 128, &pr.b, fb, n0 + 64, k);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader)
      const uint32_t idesc = idesc_bf16_f32(256, 256, true, true);
      int g = 0, n = 0;
      for (int it = cid; it < P.total; it += ncl, ++n) {
        const Item w = decode(P, it);
        const int nhi = (NH == 2 && w.tn * kTN + 256 >= P.prob[w.p].N) ? 1 : NH;
        int kb0, kb1;
        kb_range(w.slice, kb0, kb1);
        const int b = n % kNbuf;
        mbar_wait(&tempty[b], ((n / kNbuf) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + 256u * NH * (uint32_t)b;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait(&full[s], (g / kStages) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sStage + s * kStage);
          if (!(P.dbg & 2))
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks)
#pragma unroll
            for (int h = 0; h < NH; ++h)
              if (h < nhi)
              mma_pair(d + 256u * h, smem_desc_sw128(a_base + ks * 2048, kBK * 128, 1024),
                       smem_desc_sw128(a_base + kHalf * (1 + h) + ks * 2048, kBK * 128, 1024), idesc,
                       (kb != kb0 || ks != 0));
          commit_pair(&used[s]);
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[b]);
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------------------------ bias gradient (warps 6..9)
    // this CTA's dZ columns of a stage: 2 NH boxes of 64 (box bx = half bx / 2, CTA columns
    // [64 (bx & 1), +64) of it).  Lane l reads 16 bytes (8 columns: box (l % 16NH) / 8, chunk
    // l % 8 of the SW128 row) of K row RPI i + l / 16NH; warp h sums rows [RW h, RW h + RW)
    constexpr int LPR = 16 * NH, RPI = 32 / LPR;          // lanes per row, rows per instruction
    constexpr int RW = 64 / kBiasW;                       // K rows per bias warp
    const int hw = warp - 6;
    const int box = (lane % LPR) >> 3, chunk = lane & 7, rsub = lane / LPR;
    int g = 0;
    for (int it = cid; it < P.total; it += ncl) {
      const Item w = decode(P, it);
      int kb0, kb1;
      kb_range(w.slice, kb0, kb1);
      const bool do_db = w.tm == 0 && P.prob[w.p].db != nullptr && !(P.dbg & 1);
      f32x2 acc[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % kStages;
        mbar_wait(&used[s], (g / kStages) & 1);
        if (do_db) {
          const uint32_t base = smem_u32(sStage + s * kStage) + kHalf + (uint32_t)box * (kBK * 128);
#pragma unroll
          for (int i = 0; i < RW / RPI; ++i) {
            const int r = RW * hw + RPI * i + rsub;
            const uint4 v = lds128(base + (uint32_t)r * 128u + (uint32_t)((chunk ^ (r & 7)) << 4));
            const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              acc[j] = f2_add(acc[j], f2_pack(__uint_as_float(u[j] << 16), __uint_as_float(u[j] & 0xffff0000u)));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (do_db) {
        float c[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) f2_unpack(acc[j], c[2 * j], c[2 * j + 1]);
        if (RPI == 2) {
#pragma unroll
          for (int j = 0; j < 8; ++j) c[j] += __shfl_xor_sync(0xffffffffu, c[j], 16);   // rows 2 i, 2 i + 1
        }
        if (lane < LPR) {                                   // this CTA's column 8 lane .. + 7
          float4* dst4 = reinterpret_cast<float4*>(sDb + 128 * NH * hw + 8 * lane);
          dst4[0] = make_float4(c[0], c[1], c[2], c[3]);
          dst4[1] = make_float4(c[4], c[5], c[6], c[7]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kBiasW) : "memory");
        if (hw == 0) {                                    // 128 NH columns, 4 NH per lane
          const PdwProblem& pr = P.prob[w.p];
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int cl = 128 * h + 4 * lane;            // CTA column: half h, 128 per half
            float4 o = *reinterpret_cast<const float4*>(sDb + cl);
#pragma unroll
            for (int x = 1; x < kBiasW; ++x) {
              const float4 t = *reinterpret_cast<const float4*>(sDb + 128 * NH * x + cl);
              o.x += t.x; o.y += t.y; o.z += t.z; o.w += t.w;
            }
            const int col = w.tn * kTN + 256 * h + 128 * (int)rank + 4 * lane;
            float* dst = pr.db + (size_t)w.slice * (size_t)pr.db_stride + col;
            const float v[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (col + i < pr.N) dst[i] = v[i];
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kBiasW) : "memory");    // sDb reusable
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;                               // TMEM lane quarter = 32 rows of dW
    const int ew = warp - 2;
    const uint32_t stg0 = smem_u32(sStg + (size_t)ew * kNStg * kStgBuf);
    const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
    const uint32_t row_sw = (uint32_t)((lane >> 3) * 1024 + (lane & 7) * 128);
    int n = 0;
    for (int it = cid; it < P.total; it += ncl, ++n) {
      const Item w = decode(P, it);
      const PdwProblem& pr = P.prob[w.p];
      const int b = n % kNbuf;
      const int mrow0 = w.tm * 256 + 128 * (int)rank + 32 * q;
      const int ncol0 = w.tn * kTN;
      const int nch = min(kTN, pr.N - ncol0 + 63) / 64;   // 64-column chunks with data
      if (lane == 0) bulk_wait_read<0>();                 // staging of the previous item read
      __syncwarp();
      mbar_wait(&tfull[b], (n / kNbuf) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + 256u * NH * (uint32_t)b + ((uint32_t)(q * 32) << 16);
      uint32_t v[64];
      tmem_ld32_nowait(tbase, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32_nowait(tbase + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      for (int c = 0; c < nch; ++c) {
        tmem_ld_wait();
        uint32_t f[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) f[i] = v[i];
        if (c == nch - 1) {                               // accumulator(s) b free for item n + kNbuf
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_remote(tempty_leader + 8u * (uint32_t)b);
        } else {
          tmem_ld32_nowait(tbase + 64u * (uint32_t)(c + 1), *reinterpret_cast<uint32_t(*)[32]>(v));
          tmem_ld32_nowait(tbase + 64u * (uint32_t)(c + 1) + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        }
        // chunk c: fp32 columns [64 c, 64 c + 32) and [64 c + 32, 64 c + 64) in buffers
        // (2 c) % kNStg and (2 c + 1) % kNStg, free once chunk c - kNStg / 2's stores read them
        if (lane == 0 && c >= kNStg / 2) bulk_wait_read<kNStg / 2 - 1>();
        __syncwarp();
        const uint32_t b0 = stg0 + ((2 * c) % kNStg) * kStgBuf, b1 = stg0 + ((2 * c + 1) % kNStg) * kStgBuf;
        if (pr.out_t) {
          // transposed output out[n][m]: staging row = column n (32 m of this warp, 128 B), lane m
          // writes element m of every row (a conflict-free 128 B row per store instruction)
          const uint32_t moff = (uint32_t)((lane & 3) * 4), mch = (uint32_t)(lane >> 2);
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const int n = i & 31;
            const uint32_t a = (i < 32 ? b0 : b1) + (uint32_t)n * 128u + ((mch ^ (uint32_t)(n & 7)) << 4) + moff;
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(f[i]) : "memory");
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t bb = (j < 8 ? b0 : b1) + row_sw + (uint32_t)((((j & 7) ^ (lane & 7))) << 4);
            sts128(bb, make_uint4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (pr.out_t) {
            tma_store_3d(&pr.out, b0, mrow0, ncol0 + 64 * c, w.slice);
            tma_store_3d(&pr.out, b1, mrow0, ncol0 + 64 * c + 32, w.slice);
          } else {
            tma_store_3d(&pr.out, b0, ncol0 + 64 * c, mrow0, w.slice);
            tma_store_3d(&pr.out, b1, ncol0 + 64 * c + 32, mrow0, w.slice);
          }
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync();                          // the peer's MMAs / arrivals are done before TMEM goes
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// -------------------------------------------------------------------------------- host side
void pdw_init(PdwParams& P, int K, int splits, size_t split_stride) {
  P = PdwParams{};
  const char* nh = std::getenv("CRL_PDW_NH");
  P.nh = nh && std::atoi(nh) == 1 ? 1 : 2;
  P.K = K;
  P.splits = splits;
  const int nkb = (K + pdw::kBK - 1) / pdw::kBK;
  P.kb_per_split = (nkb + splits - 1) / splits;
  P.split_stride = (long long)split_stride;
}

bool pdw_supported(int K, int splits) {
  // every slice must own at least one K block (an empty slice would store a stale accumulator)
  const int nkb = (K + pdw::kBK - 1) / pdw::kBK;
  const int per = (nkb + splits - 1) / splits;
  return splits >= 1 && (long)per * (splits - 1) < nkb && !std::getenv("CRL_NO_PDW");
}

bool pdw_add_problem(PdwParams& P, const __nv_bfloat16* X, int ldx, const __nv_bfloat16* dZ, int M, int N,
                     float* dW, float* db) {
  const bool dbg = std::getenv("CRL_PDW_DEBUG") != nullptr;
  if (P.n >= kPdwMaxProblems) { if (dbg) fprintf(stderr, "pdw: table full\n"); return false; }
  if ((reinterpret_cast<uintptr_t>(dW) % 16) != 0 || (reinterpret_cast<uintptr_t>(db) % 16) != 0 || N % 4 != 0 ||
      P.split_stride % 4 != 0) {
    if (dbg) fprintf(stderr, "pdw: alignment (dW %p db %p N %d stride %lld)\n", (void*)dW, (void*)db, N, P.split_stride);
    return false;
  }
  PdwProblem& pr = P.prob[P.n];
  if (!make_map_bf16(&pr.a, X, M, P.K, ldx, 64, 64) || !make_map_bf16(&pr.b, dZ, N, P.K, N, 64, 64) ||
      !make_map_f32_3d(&pr.out, dW, N, M, P.splits, N, (uint64_t)P.split_stride, 32, 32)) {
    if (dbg) fprintf(stderr, "pdw: tensor map (M %d N %d ldx %d)\n", M, N, ldx);
    return false;
  }
  pr.db = db;
  pr.db_stride = P.split_stride;
  pr.out_t = 0;
  pr.M = M;
  pr.N = N;
  pr.tiles_n = (N + 256 * P.nh - 1) / (256 * P.nh);
  pr.tiles = ((M + 255) / 256) * pr.tiles_n * P.splits;
  P.total += pr.tiles;
  ++P.n;
  return true;
}

bool pdw_add_gemm_t(PdwParams& P, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, int ldb, int M, int N,
                    float* out_t, long long out_stride, float* colsum_b, long long colsum_stride) {
  if (P.n >= kPdwMaxProblems || (reinterpret_cast<uintptr_t>(out_t) % 16) != 0 || M % 4 != 0 || out_stride % 4 != 0 ||
      (colsum_b != nullptr && (reinterpret_cast<uintptr_t>(colsum_b) % 16) != 0))
    return false;
  PdwProblem& pr = P.prob[P.n];
  if (!make_map_bf16(&pr.a, A, M, P.K, lda, 64, 64) || !make_map_bf16(&pr.b, B, N, P.K, ldb, 64, 64) ||
      !make_map_f32_3d(&pr.out, out_t, M, N, P.splits, M, (uint64_t)out_stride, 32, 32))
    return false;
  pr.db = colsum_b;
  pr.db_stride = colsum_stride;
  pr.out_t = 1;
  pr.M = M;
  pr.N = N;
  pr.tiles_n = (N + 256 * P.nh - 1) / (256 * P.nh);
  pr.tiles = ((M + 255) / 256) * pr.tiles_n * P.splits;
  P.total += pr.tiles;
  ++P.n;
  return true;
}

void pdw_set_nh(PdwParams& P, int nh) { P.nh = nh == 1 ? 1 : 2; }

template <int NH>
static cudaError_t launch_pdw(const PdwParams& P, int num_sms, cudaStream_t st) {
  static bool attr = false;
  constexpr size_t smem = pdw::Cfg<NH>::kSmem;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_pdw_kernel<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int clusters = std::max(1, std::min(P.total, num_sms / 2));
  if (const char* d = std::getenv("CRL_PDW_DBG")) {        // measurement ablations
    PdwParams Q = P;
    Q.dbg = std::atoi(d);
    return launch_pdl(tc_pdw_kernel<NH>, dim3(2 * clusters), dim3(pdw::Cfg<NH>::kThreads), smem, st, Q);
  }
  return launch_pdl(tc_pdw_kernel<NH>, dim3(2 * clusters), dim3(pdw::Cfg<NH>::kThreads), smem, st, P);
}

cudaError_t tc_pdw_launch(const PdwParams& P, int num_sms, cudaStream_t st) {
  if (P.total == 0) return cudaSuccess;
  return P.nh == 1 ? launch_pdw<1>(P, num_sms, st) : launch_pdw<2>(P, num_sms, st);
}

}  // namespace tc
}  // namespace crl
