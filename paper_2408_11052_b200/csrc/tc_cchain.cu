// tc_cchain.cu — cluster-split MLP chains for small batches (BF16 path, width 256, D = 64).
//
// Paper: the phi / psi encoders of §3.1 P:193-195 (Table 2: hidden 256, repr 64;
// §5.4 depth 4).  Readings A-13 (SiLU), A-16 (affine output).
//
// At B_l = 256 a layer GEMM is 256 x 256 x 256: a few microseconds of latency per launch and
// almost no work.  The per-row-block chain of tc_chain.cu removes the launches but runs each
// layer on one SM per 128 rows.  Here a CLUSTER of 4 CTAs owns 128 rows: CTA c computes
// output columns [64c, 64c + 64) of every hidden layer (its slice of W: 32 KB per layer,
// streamed by TMA, the first two layers requested before the programmatic-launch wait), writes
// its 128 x 64 bf16 chunk into its own SMEM operand buffer and pushes it into the three peer
// CTAs' buffers with DSMEM bulk copies (cp.async.bulk shared::cta -> shared::cluster, signalled
// on the peers' mbarriers), so every CTA holds the full next-layer input after one exchange.
// Each chunk is also TMA-stored to HBM (the backward pass needs the activations).
//   FWD : Z_l = X_l W_l + b_l, X_{l+1} = SiLU(Z_l) (Z_l stored from registers, X_{l+1} by TMA);
//         the output layer (N = D = 64) runs on CTA 0 of the cluster: Y fp32 + bf16 and the
//         per-row statistic of bf16(Y) for the logits stage.
//   BWD : dZ_{l-1} = (dZ_l W_l^T) * SiLU'(Z_{l-1}), l = L-1 .. 1, from dY; dZ stored by TMA.
// blockIdx.y picks phi or psi: both encoders in one launch.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_cchain.h"

namespace crl {
namespace tc {

namespace cc {
constexpr uint32_t CHUNK = 128 * 128;            // 128 rows x 64 bf16 (SW128 K chunk)
constexpr uint32_t WSTAGE = 4 * 64 * 64 * 2;     // 4 K-chunks x (64 K rows x 64 N) = 32 KB
constexpr uint32_t WSTAGE0 = 5 * 64 * 64 * 2;    // stage 0 also holds a 5-chunk first layer (in0 <= 320)
constexpr int NC = 4;                            // cluster size = hidden width / 64

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// SMEM -> peer SMEM bulk copy completing on the peer's mbarrier
__device__ __forceinline__ void dsmem_copy(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
               : "memory");
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
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// mbarrier wait with cluster-scope acquire (the arrivals are remote releases)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC_%=;\n\t"
      "bra WAITC_%=;\n"
      "DONEC_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
}  // namespace cc

template <int MODE>   // 0 = forward, 1 = backward dX chain
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(384, 1)
    tc_cchain_kernel(const __grid_constant__ CChainMaps maps0, const __grid_constant__ CChainMaps maps1,
                     const CChainParams p) {
  using namespace cc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAct = smem;                                        // [2][4] chunks (layer-parity buffers)
  uint8_t* sX4 = sAct + 2 * NC * CHUNK;                        // 5th K chunk of a wide first-layer input
  uint8_t* sW = sX4 + CHUNK;                                   // weight stages: 0 (40 KB), 1 (32 KB)
  float* sBias = reinterpret_cast<float*>(sW + WSTAGE0 + WSTAGE);   // [kCChainMaxL][64]
  float* sStat = sBias + kCChainMaxL * 64;                     // [128] row-stat hand-off
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStat + 128);
  uint64_t* a0_full = bars;                 // first-layer input (from HBM) in act buffer 0
  uint64_t* in_full = bars + 1;             // [2][4] next-layer input chunk j arrived (per source CTA)
  uint64_t* w_full = in_full + 2 * NC;      // [2]
  uint64_t* w_empty = w_full + 2;           // [2]
  uint64_t* acc_full = w_empty + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);

  const int enc = blockIdx.y;
  const CChainMaps& mp = enc ? maps1 : maps0;
  const CChainEnc& E = p.enc[enc];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = cluster_rank();                           // this CTA's 64-column slice
  const int m0 = (blockIdx.x / NC) * 128;
  const int L = E.L;                                           // GEMM steps of this encoder

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mp.a0);
    mbar_init(a0_full, 1);
    for (int i = 0; i < 2; ++i) {
      for (int j = 0; j < NC; ++j) mbar_init(&in_full[i * NC + j], 1);   // leader arrival (+ peer bytes)
      mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1);
      mbar_init(&acc_full[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  cluster_sync();                          // every CTA's barriers exist before peers signal them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // step s computes a slice of every CTA except the FWD output layer (CTA 0 only)
  auto active = [&](int s) { return !(MODE == 0 && s == L - 1) || c == 0; };
  auto load_w = [&](int s) {
    const CChainLayer& Ly = E.layer[s];
    const int st = s & 1;
    const int nkc = (Ly.K + 63) / 64;
    mbar_expect_tx(&w_full[st], (uint32_t)nkc * 8192u);
    const int n0 = (MODE == 0 && s == L - 1) ? 0 : 64 * (int)c;
    for (int kc = 0; kc < nkc; ++kc)
      // FWD: W_l [in][out] MN-major slice, box {64 (out), 64 (in)} at (n0, 64 kc)
      // BWD: W_l rows n0.. as the K-major B of dZ W^T, box {64 (out = k), 64 (in = n)}
      tma_load_2d(sW + (st ? WSTAGE0 : 0u) + kc * 8192, &mp.w[s], &w_full[st], MODE == 0 ? n0 : 64 * kc,
                  MODE == 0 ? 64 * kc : n0);
  };
  // the weights do not depend on the predecessor kernel: request the first two layers now
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 2 && s < L; ++s)
      if (active(s)) load_w(s);
  }
  if (MODE == 0 && warp >= 4) {                              // bias slices of this CTA
    for (int i = threadIdx.x - 128; i < L * 64; i += 256) {
      const int s = i / 64, j = i % 64;
      const int col = (s == L - 1) ? j : 64 * (int)c + j;
      sBias[i] = (s < L && col < E.layer[s].N) ? E.layer[s].bias[col] : 0.f;
    }
  }
  __shared__ unsigned long long s_tt[24];
  const bool trace = p.trace && blockIdx.x == 0 && blockIdx.y == 0;
  auto gt = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  if (trace && threadIdx.x == 0) s_tt[0] = gt();
  pdl_wait();
  pdl_launch();
  if (trace && threadIdx.x == 0) s_tt[1] = gt();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------------ TMA producer
    const int nch0 = (E.layer[0].K + 63) / 64;
    mbar_expect_tx(a0_full, (uint32_t)nch0 * CHUNK);
    for (int k = 0; k < nch0; ++k) tma_load_2d(k < NC ? sAct + k * CHUNK : sX4, &mp.a0, a0_full, 64 * k, m0);
    for (int s = 2; s < L; ++s) {
      if (!active(s)) continue;
      mbar_wait(&w_empty[s & 1], ((s >> 1) - 1) & 1);
      load_w(s);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ MMA issuer
    for (int s = 0; s < L; ++s) {
      if (!active(s)) break;
      const CChainLayer& Ly = E.layer[s];
      const int nkc = (Ly.K + 63) / 64;
      const uint32_t acc = tmem + (uint32_t)((s & 1) * 64);
      // input of step s: HBM tile (s = 0) or the exchanged chunks (buffer s & 1), consumed in
      // arrival order: this CTA's own chunk first, then the peers' as their copies land
      if (s == 0) mbar_wait(a0_full, 0);
      mbar_wait(&w_full[s & 1], (s >> 1) & 1);
      const uint32_t a_base = smem_u32(sAct + (s & 1) * NC * CHUNK);
      const uint32_t w_base = smem_u32(sW + ((s & 1) ? WSTAGE0 : 0u));
      const uint32_t idesc = idesc_bf16_f32(128, 64, false, MODE == 0);
      for (int i = 0; i < nkc; ++i) {
        const int kc = s == 0 ? i : (int)((c + i) % NC);
        if (s > 0) {
          mbar_wait_cluster(&in_full[(s & 1) * NC + kc], ((s - 1) >> 1) & 1);
          // written by (remote) generic-proxy stores, read by the tensor core (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t a_chunk = (s == 0 && kc == NC) ? smem_u32(sX4) : a_base + kc * CHUNK;
          const uint64_t ad = smem_desc_sw128(a_chunk + ks * 32, 16, 1024);
          const uint64_t bd = MODE == 0 ? smem_desc_sw128(w_base + kc * 8192 + ks * 2048, 8192, 1024)
                                        : smem_desc_sw128(w_base + kc * 8192 + ks * 32, 16, 1024);
          mma_bf16(acc, ad, bd, idesc, (i | ks) != 0);
        }
        if (trace && s < 6 && i == 0) s_tt[12 + 2 * s] = gt();      // first chunk issued
        if (trace && s < 6 && i == nkc - 1) s_tt[13 + 2 * s] = gt(); // last chunk issued
      }
      mma_commit(&acc_full[s & 1]);
      mma_commit(&w_empty[s & 1]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue (2 warpgroups)
    const int wg = (warp - 4) >> 2;                 // 32 of the slice's 64 columns
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int row = m0 + r;
    const bool rv = row < p.M;
    const bool leader = wg == 0 && q == 0 && lane == 0;
    const uint32_t row_off = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    for (int s = 0; s < L; ++s) {
      if (!active(s)) break;
      const CChainLayer& Ly = E.layer[s];
      const bool last_fwd = MODE == 0 && s == L - 1;
      const bool last_bwd = MODE == 1 && s == L - 1;
      const int col0 = (last_fwd ? 0 : 64 * (int)c) + 32 * wg;      // global output column
      uint4 zp[4];                                   // BWD: Z_{l-1} of these 32 columns (bf16)
      if (MODE == 1 && rv) {
        const uint4* zr = reinterpret_cast<const uint4*>(Ly.zprev + (size_t)row * Ly.N + col0);
#pragma unroll
        for (int j = 0; j < 4; ++j) zp[j] = zr[j];
      }
      mbar_wait(&acc_full[s & 1], (s >> 1) & 1);
      if (trace && leader && s < 10) s_tt[2 + 2 * s] = gt();
      tc_fence_after();
      uint32_t raw[32];
      tmem_ld32_nowait(tmem + (uint32_t)((s & 1) * 64) + ((uint32_t)(q * 32) << 16) + 32 * wg, raw);
      tmem_ld_wait();
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
      if (MODE == 0) {                               // bias: 8 vector shared loads
        const uint32_t ba = smem_u32(sBias + s * 64 + 32 * wg);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 b;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                       : "r"(ba + 16u * j));
          v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
        }
      }
      if (last_fwd) {
        // Y fp32 + bf16 and the row statistic of bf16(Y) (CTA 0 holds the whole row)
        float ysq = 0.f;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
          const float2 yb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[i]));
          ysq = fmaf(yb.x, yb.x, fmaf(yb.y, yb.y, ysq));
        }
        if (rv) {
          float4* yf = reinterpret_cast<float4*>(Ly.out_f + (size_t)row * Ly.N + col0);
#pragma unroll
          for (int i = 0; i < 8; ++i) yf[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          uint4* yb = reinterpret_cast<uint4*>(Ly.out_act + (size_t)row * Ly.N + col0);
#pragma unroll
          for (int i = 0; i < 4; ++i) yb[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
        if (wg == 1) sStat[r] = ysq;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (wg == 0 && rv && E.out_stat != nullptr) {
          const float st = ysq + sStat[r];
          E.out_stat[row] = (p.energy == CRL_ENERGY_L2 || p.energy == CRL_ENERGY_L2SQ) ? st
                            : (p.energy == CRL_ENERGY_COS ? 1.f / fmaxf(sqrtf(st), kEpsCos) : 0.f);
        }
        break;
      }
      uint32_t pk[16];                               // bf16 pairs of the chunk value
      if (MODE == 0) {
        uint32_t zk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          zk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
          float a0, a1;
          if (p.act == CRL_ACT_SILU) {
            const float h0 = 0.5f * v[2 * i], h1 = 0.5f * v[2 * i + 1];
            a0 = fmaf(h0, tanh_fast(h0), h0);
            a1 = fmaf(h1, tanh_fast(h1), h1);
          } else {
            a0 = fmaxf(v[2 * i], 0.f);
            a1 = fmaxf(v[2 * i + 1], 0.f);
          }
          pk[i] = pack_bf16x2(a0, a1);
        }
        if (rv && p.store_ok) {                      // Z_l: 64 contiguous bytes of the row
          uint4* zo = reinterpret_cast<uint4*>(Ly.out_z + (size_t)row * Ly.N + col0);
#pragma unroll
          for (int i = 0; i < 4; ++i) zo[i] = make_uint4(zk[4 * i], zk[4 * i + 1], zk[4 * i + 2], zk[4 * i + 3]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t zw = reinterpret_cast<const uint32_t*>(zp)[i];
          const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zw));
          float g0, g1;
          if (p.act == CRL_ACT_SILU) {
            const float h0 = 0.5f * z.x, h1 = 0.5f * z.y;
            const float t0 = tanh_fast(h0), t1 = tanh_fast(h1);
            g0 = fmaf(0.5f, fmaf(h0, fmaf(-t0, t0, 1.f), t0), 0.5f);
            g1 = fmaf(0.5f, fmaf(h1, fmaf(-t1, t1, 1.f), t1), 0.5f);
          } else {
            g0 = z.x > 0.f ? 1.f : 0.f;
            g1 = z.y > 0.f ? 1.f : 0.f;
          }
          pk[i] = pack_bf16x2(v[2 * i] * g0, v[2 * i + 1] * g1);
        }
      }
      // the chunk (this CTA's 64 columns of the next-layer input) -> own SMEM buffer, then one
      // DSMEM bulk copy to each peer.  (Measured alternative: every thread storing its rows
      // into the peers with st.shared::cluster is 3x slower per step on B200.)
      const int nb = (s + 1) & 1;
      uint8_t* chunk = sAct + nb * NC * CHUNK + c * CHUNK;
      const uint32_t dst = smem_u32(chunk) + row_off;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 32 * wg + 8 * u;
        sts128(dst + (uint32_t)((((k >> 3) ^ (r & 7))) << 4),
               rv ? make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]) : make_uint4(0u, 0u, 0u, 0u));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (leader) {
        // the FWD output layer runs on CTA 0 only: the others neither need nor wait for its
        // input, and must not receive copies they will never wait for
        const bool to_last = MODE == 0 && s + 1 == L - 1;
        if (!last_bwd) {
          const uint32_t src = smem_u32(chunk);
          const uint32_t bar_local = smem_u32(&in_full[nb * NC + c]);   // "chunk c arrived"
#pragma unroll
          for (int i = 1; i < NC; ++i) {
            const uint32_t peer = (c + i) % NC;
            if (to_last && peer != 0) continue;
            dsmem_copy(mapa(src, peer), src, CHUNK, mapa(bar_local, peer));
          }
        }
        if (p.store_ok) {                            // HBM copy (X_{l+1} or dZ_{l-1})
          tma_store_2d(&mp.st[s], smem_u32(chunk), 64 * (int)c, m0);
          bulk_commit();
        }
        // The other buffer is rewritten by the NEXT step's epilogue, which can only start after
        // the next MMA, which waits for this CTA's arrival below: the HBM store issued one step
        // ago from that buffer must have read it by then (at most this step's store pending).
        // (Peer copies are covered by causality: the peers consumed the buffer before that.)
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (!last_bwd && (!to_last || c == 0)) {
          // the peers' chunks: expect their bytes; this CTA's own chunk: plain arrival
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            if (j == (int)c) mbar_arrive(&in_full[nb * NC + j]);
            else mbar_expect_tx(&in_full[nb * NC + j], CHUNK);
          }
        }
        if (trace && s < 10) s_tt[3 + 2 * s] = gt();
      }
    }
    if (leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                          // no CTA leaves while a peer may still copy into it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
  if (trace && threadIdx.x == 0) {
    printf("CCHAIN_TRACE mode=%d L=%d pdl_wait=%llu", MODE, L, s_tt[1] - s_tt[0]);
    for (int s = 0; s < L && s < 5; ++s)
      printf(" | s%d mma0=%llu mmaN=%llu acc=%llu done=%llu", s, s_tt[12 + 2 * s] - s_tt[0], s_tt[13 + 2 * s] - s_tt[0],
             s_tt[2 + 2 * s] - s_tt[0], s_tt[3 + 2 * s] - s_tt[0]);
    printf(" | end=%llu\n", gt() - s_tt[0]);
  }
}

size_t tc_cchain_smem() {
  return 1024 + (2 * cc::NC + 1) * cc::CHUNK + cc::WSTAGE0 + cc::WSTAGE + kCChainMaxL * 64 * 4 + 512 + 256;
}

bool tc_cchain_supported(int in0, int width, int D, int depth) {
  return width == 256 && D == 64 && in0 <= 320 && depth >= 1 && depth + 1 <= kCChainMaxL;
}

template <int MODE>
static cudaError_t launch_cchain(const CChainMaps& m0, const CChainMaps& m1, const CChainParams& p, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = tc_cchain_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_cchain_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(cc::NC * ((p.M + 127) / 128), 2);
  return launch_pdl(tc_cchain_kernel<MODE>, grid, dim3(384), smem, st, m0, m1, p);
}

cudaError_t tc_cchain_forward(const CChainMaps& m0, const CChainMaps& m1, const CChainParams& p, cudaStream_t st) {
  return launch_cchain<0>(m0, m1, p, st);
}
cudaError_t tc_cchain_backward(const CChainMaps& m0, const CChainMaps& m1, const CChainParams& p, cudaStream_t st) {
  return launch_cchain<1>(m0, m1, p, st);
}

}  // namespace tc
}  // namespace crl
