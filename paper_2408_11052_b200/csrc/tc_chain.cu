// tc_chain.cu — fused per-row-block MLP chains on tcgen05 (BF16 path, width <= 256).
//
// Paper: §3.1 P:193-195 (phi(s,a), psi(g)), Table 2 P:943-944 (hidden [256,256], repr 64),
// §5.4 (depth 4).  Readings A-13 (SiLU), A-16 (affine output).
//
// One CTA owns 128 rows of the batch and runs EVERY layer of one encoder (blockIdx.y picks
// phi or psi, so both encoders run in one launch).  Activations never leave the SM between
// layers: layer l's epilogue writes its bf16 output straight into the SMEM operand buffer
// (SW128 K-major, one 16 KB chunk per 64 features) that layer l+1's tcgen05.mma reads, and
// the same SMEM chunk is written to HBM by one TMA bulk-tensor store (the activations are
// needed again by the backward pass) — coalesced and asynchronous, instead of row-per-thread
// global stores.  Pipelining: the TMEM accumulator is double-buffered and every 64-feature
// chunk is handed to the MMA warp as soon as it is written (act_ready[c]), so layer l+1's
// MMAs overlap layer l's epilogue; two epilogue warpgroups split the columns; the weights
// stream through a TMA ring that runs ahead across layer boundaries.
//   FWD : Z_l = X_l W_l + b_l, X_{l+1} = SiLU(Z_l) (Z_l, X_{l+1} stored for backward);
//         output Y (fp32 + bf16) and the per-row statistic of the bf16 Y used by the logits
//         stage (L2: |y|^2, cos: 1/max(|y|, eps)).
//   BWD : dZ_{l-1} = (dZ_l W_l^T) * SiLU'(Z_{l-1}) for l = L-1 .. 1, starting from dY;
//         every dZ is stored for the dW / db reductions.
// SiLU uses sigmoid(z) = (1 + tanh(z/2)) / 2 with the tanh.approx MUFU op (one MUFU op per
// element instead of exp + reciprocal); the path's tolerance is 2e-2 (north_star).
#include <cstdio>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_chain.h"

namespace crl {
namespace tc {

// Weight K-block stages and store staging per mode (same SMEM total): the forward stages Z_l /
// Y for TMA stores (4 chunks) and keeps 2 weight stages; the backward has no staging and keeps
// 4 weight stages = a whole 256-wide layer, so the next layer's weights are requested before
// this layer's dZ stores enter the SM's TMA queue (measured: 2 stages put the last two
// blocks ~4000 clk behind the stores; backward 66 -> 63 us at N = 16384.  Direct-from-register
// Z stores in the forward, to free room for 4 stages there, were slower: 66 -> 72 us)
template <int MODE> struct ChCfg {
  static constexpr int STAGES = MODE == 0 ? 2 : 4;
  static constexpr int STG_CHUNKS = MODE == 0 ? 4 : 0;
};
constexpr int CH_ACT_CHUNKS = 5;                  // K <= 320
constexpr uint32_t CH_CHUNK = 128 * 128;          // 128 rows x 64 bf16 (one SW128 K chunk)
constexpr uint32_t CH_WSTAGE = 64 * 256 * 2;      // 64 K rows x up to 256 N
constexpr int CH_BIAS = kChainMaxL * 256;

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void wg_sync(int wg) { asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory"); }
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// silu(z) = z sigmoid(z) = h + h tanh(h), h = z/2
__device__ __forceinline__ float silu_fast(float z) {
  const float h = 0.5f * z;
  return fmaf(h, tanh_approx(h), h);
}
// silu'(z) = s (1 + z (1 - s)) = 1/2 + (t + h (1 - t^2)) / 2, t = tanh(h), h = z/2
__device__ __forceinline__ float silu_grad_fast(float z) {
  const float h = 0.5f * z;
  const float t = tanh_approx(h);
  return fmaf(0.5f, fmaf(h, fmaf(-t, t, 1.f), t), 0.5f);
}
// FWD hidden layer: Z = acc + b (bf16 pairs zk), X' = act(Z) (bf16 pairs pk)
template <bool SILU, int NE>
__device__ __forceinline__ void epi_fwd_hidden(uint32_t* raw, uint32_t bias_a, uint32_t* pk, uint32_t* zk) {
#pragma unroll
  for (int j = 0; j < NE / 4; ++j) {
    const float4 b = lds128f(bias_a + 16u * j);
    const float z0 = __uint_as_float(raw[4 * j]) + b.x, z1 = __uint_as_float(raw[4 * j + 1]) + b.y;
    const float z2 = __uint_as_float(raw[4 * j + 2]) + b.z, z3 = __uint_as_float(raw[4 * j + 3]) + b.w;
    zk[2 * j] = pack_bf16x2(z0, z1);
    zk[2 * j + 1] = pack_bf16x2(z2, z3);
    if (SILU) {
      pk[2 * j] = pack_bf16x2(silu_fast(z0), silu_fast(z1));
      pk[2 * j + 1] = pack_bf16x2(silu_fast(z2), silu_fast(z3));
    } else {
      pk[2 * j] = pack_bf16x2(fmaxf(z0, 0.f), fmaxf(z1, 0.f));
      pk[2 * j + 1] = pack_bf16x2(fmaxf(z2, 0.f), fmaxf(z3, 0.f));
    }
  }
}
// FWD output layer: Y = acc + b (fp32 back into raw, bf16 pairs pk); returns sum of bf16(Y)^2
template <int NE>
__device__ __forceinline__ float epi_fwd_last(uint32_t* raw, uint32_t bias_a, uint32_t* pk) {
  float st = 0.f;
#pragma unroll
  for (int j = 0; j < NE / 4; ++j) {
    const float4 b = lds128f(bias_a + 16u * j);
    const float y0 = __uint_as_float(raw[4 * j]) + b.x, y1 = __uint_as_float(raw[4 * j + 1]) + b.y;
    const float y2 = __uint_as_float(raw[4 * j + 2]) + b.z, y3 = __uint_as_float(raw[4 * j + 3]) + b.w;
    raw[4 * j] = __float_as_uint(y0); raw[4 * j + 1] = __float_as_uint(y1);
    raw[4 * j + 2] = __float_as_uint(y2); raw[4 * j + 3] = __float_as_uint(y3);
    pk[2 * j] = pack_bf16x2(y0, y1);
    pk[2 * j + 1] = pack_bf16x2(y2, y3);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[2 * j]));
    const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[2 * j + 1]));
    st = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(c.x, c.x, fmaf(c.y, c.y, st))));
  }
  return st;
}
// BWD: dZ_{l-1} = acc * act'(Z_{l-1})
template <bool SILU, int NE>
__device__ __forceinline__ void epi_bwd(const uint32_t* raw, const uint32_t* zw, uint32_t* pk) {
#pragma unroll
  for (int i = 0; i < NE / 2; ++i) {
    const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zw[i]));
    const float g0 = SILU ? silu_grad_fast(z.x) : (z.x > 0.f ? 1.f : 0.f);
    const float g1 = SILU ? silu_grad_fast(z.y) : (z.y > 0.f ? 1.f : 0.f);
    pk[i] = pack_bf16x2(__uint_as_float(raw[2 * i]) * g0, __uint_as_float(raw[2 * i + 1]) * g1);
  }
}

constexpr int CH_NWG = 4;                        // epilogue warpgroups: one 64-feature chunk each
constexpr int CH_NT = 128 + 128 * CH_NWG;

template <int MODE>   // 0 = forward, 1 = backward dX chain
__global__ void __launch_bounds__(CH_NT, 1) tc_chain_kernel(const __grid_constant__ ChainMaps maps0,
                                                          const __grid_constant__ ChainMaps maps1,
                                                          const ChainParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAct = smem;
  uint8_t* sStg = sAct + CH_ACT_CHUNKS * CH_CHUNK;
  constexpr int CH_STAGES = ChCfg<MODE>::STAGES;
  uint8_t* sW = sStg + ChCfg<MODE>::STG_CHUNKS * CH_CHUNK;
  float* sBias = reinterpret_cast<float*>(sW + CH_STAGES * CH_WSTAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBias + CH_BIAS);
  uint64_t* a0_full = bars;
  uint64_t* w_full = bars + 1;
  uint64_t* w_empty = w_full + CH_STAGES;
  uint64_t* acc_full = w_empty + CH_STAGES;           // [2] per TMEM buffer
  uint64_t* act_ready = acc_full + 2;                 // [CH_ACT_CHUNKS] per 64-feature chunk
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_ready + CH_ACT_CHUNKS);

  const int enc = blockIdx.y;
  const ChainMaps& mp = enc ? maps1 : maps0;
  const ChainEnc& E = p.enc[enc];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int L = E.L;
  // dbg & 4: clock64 trace of CTA (0,0) printed at exit (measurement only)
  __shared__ long long s_tr[64];
  const bool trace = (p.dbg & 4) && blockIdx.x == 0 && blockIdx.y == 0;
#define CH_TR(i) do { if (trace) s_tr[(i)] = clock64(); } while (0)
  // row blocks walk the K blocks of each layer from staggered starts (dbg & 8 disables): in
  // lockstep every CTA fetches the same weight block from the same L2 lines at once
  // (measured at N = 16384: forward 66 -> 63 us, backward unchanged)
  const int rot = (p.dbg & 8) ? 0 : (int)blockIdx.x;
  auto kb_rot = [&](int i, int n) { return (i + rot) % n; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mp.a0);
    mbar_init(a0_full, 1);
    for (int s = 0; s < CH_STAGES; ++s) { mbar_init(&w_full[s], 1); mbar_init(&w_empty[s], 1); }
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    for (int c = 0; c < CH_ACT_CHUNKS; ++c) mbar_init(&act_ready[c], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) CH_TR(0);
  if (MODE == 0 && p.fac_ok != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    *p.fac_ok = p.fac_init;

  if (warp == 0 && lane == 0) {
    // -------------------------------------------------------------------- TMA producer
    const int nch0 = (E.layer[0].K + 63) / 64;
    mbar_expect_tx(a0_full, nch0 * CH_CHUNK);
    for (int c = 0; c < nch0; ++c) tma_load_2d(sAct + c * CH_CHUNK, &mp.a0, a0_full, 64 * c, m0);
    int g = 0;
    for (int l = 0; l < L; ++l) {
      const ChainLayer& Ly = E.layer[l];
      const int nkb = (Ly.K + 63) / 64;
      const uint32_t bytes = 64u * Ly.N * 2u;
      for (int kbi = 0; kbi < nkb; ++kbi, ++g) {
        const int kb = kb_rot(kbi, nkb);
        const int s = g % CH_STAGES;
        mbar_wait(&w_empty[s], ((g / CH_STAGES) & 1) ^ 1);
        if (g < 20) CH_TR(1 + g);
        mbar_expect_tx(&w_full[s], bytes);
        uint8_t* dst = sW + s * CH_WSTAGE;
        if (MODE == 0) {
          for (int c = 0; c < Ly.N / 64; ++c) tma_load_2d(dst + c * 8192, &mp.w[l], &w_full[s], 64 * c, 64 * kb);
        } else {
          tma_load_2d(dst, &mp.w[l], &w_full[s], 64 * kb, 0);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // -------------------------------------------------------------------- MMA issuer
    const uint32_t act_base = smem_u32(sAct);
    int g = 0;
    for (int l = 0; l < L; ++l) {
      const ChainLayer& Ly = E.layer[l];
      const uint32_t acc = tmem + (uint32_t)((l & 1) * 256);
      const uint32_t idesc = idesc_bf16_f32(128, Ly.N, false, MODE == 0);
      const int nkb = (Ly.K + 63) / 64;
      if (l == 0) mbar_wait(a0_full, 0);
      for (int kbi = 0; kbi < nkb; ++kbi, ++g) {
        const int kb = kb_rot(kbi, nkb);
        if (l > 0) mbar_wait(&act_ready[kb], (l - 1) & 1);   // chunk kb of this layer's input
        const int s = g % CH_STAGES;
        mbar_wait(&w_full[s], (g / CH_STAGES) & 1);
        if (g < 20) CH_TR(21 + g);
        tc_fence_after();
        const uint32_t wb = smem_u32(sW + s * CH_WSTAGE);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = smem_desc_sw128(act_base + kb * CH_CHUNK + ks * 32, 16, 1024);
          const uint64_t bd = MODE == 0 ? smem_desc_sw128(wb + ks * 2048, 8192, 1024)
                                        : smem_desc_sw128(wb + ks * 32, 16, 1024);
          mma_bf16(acc, ad, bd, idesc, (kbi | ks) != 0);
        }
        mma_commit(&w_empty[s]);
      }
      mma_commit(&acc_full[l & 1]);
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------------- epilogue (4 warpgroups)
    // warpgroup wg owns the 64-feature chunks c = wg, wg + 4, ... of every layer output and
    // handles each as two 32-column halves (register budget of 640 threads)
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int row = m0 + r;
    const bool rv = row < p.M;
    const bool storer = (q == 0 && lane == 0);          // issues this warpgroup's TMA stores
    const bool st_ok = !(p.dbg & 1);
    const uint32_t row_a = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    if (MODE == 0) {                                   // all biases of this encoder -> SMEM
      for (int l = 0; l < L; ++l)
        for (int c = threadIdx.x - 128; c < E.layer[l].N; c += 128 * CH_NWG) sBias[l * 256 + c] = E.layer[l].bias[c];
      asm volatile("bar.sync 1, %0;" ::"n"(128 * CH_NWG) : "memory");
    }
    float stat = 0.f;
    for (int l = 0; l < L; ++l) {
      const ChainLayer& Ly = E.layer[l];
      const bool last = l == L - 1;
      const int N = Ly.N;
      const int nch = N / 64;
      const uint32_t acc = tmem + (uint32_t)((l & 1) * 256);
      mbar_wait(&acc_full[l & 1], (l >> 1) & 1);
      if (storer && l < 5 && wg < 2) CH_TR(42 + 5 * wg + l);
      tc_fence_after();
      // SMEM chunks are about to be rewritten: the previous layer's TMA stores (of any
      // warpgroup: the chunk owners change with N) must have read them
      if (storer) bulk_wait_read();
      asm volatile("bar.sync 1, %0;" ::"n"(128 * CH_NWG) : "memory");
      for (int c = wg; c < nch; c += CH_NWG) {
        const uint32_t bias_c = smem_u32(sBias) + (uint32_t)(l * 256 + 64 * c) * 4u;
        const uint32_t act_a = smem_u32(((MODE == 0 && last) ? sStg : sAct) + c * CH_CHUNK) + row_a;
        const uint32_t z_a = smem_u32(sStg + c * CH_CHUNK) + row_a;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {                 // 32-column halves of the chunk
          uint4 zp[4];                                   // BWD: Z_{l-1} row, these 32 features
          if (MODE == 1 && rv) {
            const uint4* zr = reinterpret_cast<const uint4*>(Ly.zprev + (size_t)row * N + 64 * c + 32 * hf);
#pragma unroll
            for (int j = 0; j < 4; ++j) zp[j] = zr[j];
          }
          uint32_t raw[32];
          tmem_ld32_nowait(acc + ((uint32_t)(q * 32) << 16) + 64 * c + 32 * hf, raw);
          tmem_ld_wait();
          uint32_t pk[16];                               // bf16 pairs of the value feeding the next step
          const uint32_t bias_a = bias_c + 128u * hf;
          if (MODE == 0 && !last) {
            uint32_t zk[16];                             // bf16 pairs of Z
            if (p.act == CRL_ACT_SILU) epi_fwd_hidden<true, 32>(raw, bias_a, pk, zk);
            else epi_fwd_hidden<false, 32>(raw, bias_a, pk, zk);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              sts128(z_a + (uint32_t)(((u + 4 * hf) ^ (r & 7)) << 4),
                     make_uint4(zk[4 * u], zk[4 * u + 1], zk[4 * u + 2], zk[4 * u + 3]));
          } else if (MODE == 0) {
            stat += epi_fwd_last<32>(raw, bias_a, pk);
          } else {
            const uint32_t* zw = reinterpret_cast<const uint32_t*>(zp);
            if (p.act == CRL_ACT_SILU) epi_bwd<true, 32>(raw, zw, pk);
            else epi_bwd<false, 32>(raw, zw, pk);
          }
          // SMEM: pk -> the operand chunk (next step's A, also the TMA-store source); FWD
          // hidden: Z -> the staging chunk (above); FWD last: Y bf16 -> staging, Y fp32 -> HBM
#pragma unroll
          for (int u = 0; u < 4; ++u)
            sts128(act_a + (uint32_t)(((u + 4 * hf) ^ (r & 7)) << 4),
                   rv ? make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]) : make_uint4(0u, 0u, 0u, 0u));
          if (MODE == 0 && last && rv && st_ok) {
            float4* yo = reinterpret_cast<float4*>(Ly.out_f + (size_t)row * N + 64 * c + 32 * hf);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              yo[u] = make_float4(__uint_as_float(raw[4 * u]), __uint_as_float(raw[4 * u + 1]),
                                  __uint_as_float(raw[4 * u + 2]), __uint_as_float(raw[4 * u + 3]));
          }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (!(MODE == 0 && last) && lane == 0) mbar_arrive(&act_ready[c]);
        // whole 128 x 64 chunk written by the 4 warps -> one TMA store per tensor
        wg_sync(wg);
        if (storer && st_ok) {
          if (MODE == 0 && !last) {
            tma_store_2d(&mp.st_out[l], sAct + c * CH_CHUNK, 64 * c, m0);
            tma_store_2d(&mp.st_z[l], sStg + c * CH_CHUNK, 64 * c, m0);
          } else if (MODE == 0) {
            tma_store_2d(&mp.st_out[l], sStg + c * CH_CHUNK, 64 * c, m0);
          } else {
            tma_store_2d(&mp.st_out[l], sAct + c * CH_CHUNK, 64 * c, m0);
          }
          bulk_commit();
        }
      }
      if (storer && wg == 0 && l < 5) CH_TR(52 + l);
    }
    if (storer) bulk_wait_all();
    if (storer && wg == 0) CH_TR(57);
    if (MODE == 0) {
      // row statistic of Y: warpgroups 1.. hand their columns' partial sums to warpgroup 0
      float* sStat = sBias;                            // biases are no longer needed
      asm volatile("bar.sync 1, %0;" ::"n"(128 * CH_NWG) : "memory");
      if (wg > 0) sStat[(wg - 1) * 128 + r] = stat;
      asm volatile("bar.sync 1, %0;" ::"n"(128 * CH_NWG) : "memory");
      if (wg == 0 && rv && E.out_stat != nullptr) {
        float st = stat;
        for (int w = 1; w < CH_NWG; ++w) st += sStat[(w - 1) * 128 + r];
        E.out_stat[row] = (p.energy == CRL_ENERGY_L2 || p.energy == CRL_ENERGY_L2SQ) ? st
                          : (p.energy == CRL_ENERGY_COS ? 1.f / fmaxf(sqrtf(st), kEpsCos) : 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (trace && threadIdx.x == 0) {
    printf("CHAIN_TRACE mode=%d L=%d\n", MODE, L);
    for (int i = 1; i < 64; ++i) printf("CHAIN_TRACE %d %lld\n", i, s_tr[i] - s_tr[0]);
  }
#undef CH_TR
}

size_t tc_chain_smem() {
  static_assert(ChCfg<0>::STG_CHUNKS * CH_CHUNK + ChCfg<0>::STAGES * CH_WSTAGE ==
                ChCfg<1>::STG_CHUNKS * CH_CHUNK + ChCfg<1>::STAGES * CH_WSTAGE, "one SMEM size for both modes");
  return 1024 + (CH_ACT_CHUNKS + ChCfg<0>::STG_CHUNKS) * CH_CHUNK + ChCfg<0>::STAGES * CH_WSTAGE + CH_BIAS * 4 + 256;
}

bool tc_chain_supported(int in0, int width, int D, int depth) {
  return depth + 1 <= kChainMaxL && width <= 256 && width % 64 == 0 && D % 64 == 0 && D <= 256 &&
         in0 <= CH_ACT_CHUNKS * 64;
}

template <int MODE>
static cudaError_t launch_chain(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, int nenc,
                                cudaStream_t st) {
  static bool attr = false;
  const size_t smem = tc_chain_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_chain_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.M + 127) / 128, nenc);
  return launch_pdl(tc_chain_kernel<MODE>, grid, dim3(CH_NT), smem, st, m0, m1, p);
}

cudaError_t tc_chain_forward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st) {
  return launch_chain<0>(m0, m1, p, 2, st);
}
cudaError_t tc_chain_backward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st) {
  return launch_chain<1>(m0, m1, p, 2, st);
}

}  // namespace tc
}  // namespace crl
