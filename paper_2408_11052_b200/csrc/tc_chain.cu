// tc_chain.cu — fused per-row-block MLP chains on tcgen05 (BF16 path, width <= 256).
//
// Paper: §3.1 P:193-195 (phi(s,a), psi(g)), Table 2 P:943-944 (hidden [256,256], repr 64),
// §5.4 (depth 4).  Readings A-13 (SiLU), A-16 (affine output).
//
// One CTA owns 128 rows of the batch and runs EVERY layer of one encoder (blockIdx.y picks
// phi or psi, so both encoders run in one launch).  Activations never leave the SM between
// layers: layer l's epilogue writes its bf16 output straight into the SMEM operand buffer
// (SW128 K-major, one 16 KB chunk per 64 features) that layer l+1's tcgen05.mma reads.
// Pipelining: the TMEM accumulator is double-buffered and every 64-feature chunk is handed
// to the MMA warp as soon as it is written (act_ready[c]), so layer l+1's MMAs overlap layer
// l's epilogue; two epilogue warpgroups split the columns of each layer; the weights stream
// through a 3-stage TMA ring that runs ahead across layer boundaries.
//   FWD : Z_l = X_l W_l + b_l, X_{l+1} = SiLU(Z_l) (Z_l, X_{l+1} also stored for backward);
//         output Y (fp32 + bf16) and the per-row statistic of the bf16 Y used by the logits
//         stage (L2: |y|^2, cos: 1/max(|y|, eps)).
//   BWD : dZ_{l-1} = (dZ_l W_l^T) * SiLU'(Z_{l-1}) for l = L-1 .. 1, starting from dY;
//         every dZ is stored for the dW / db reductions.
// SiLU uses sigmoid(z) = (1 + tanh(z/2)) / 2 with the tanh.approx MUFU op (one MUFU op per
// element instead of exp + reciprocal); the path's tolerance is 2e-2 (north_star).
#include "common.cuh"
#include "tc_common.cuh"
#include "tc_chain.h"

namespace crl {
namespace tc {

constexpr int CH_STAGES = 3;
constexpr int CH_ACT_CHUNKS = 5;                  // K <= 320
constexpr uint32_t CH_CHUNK = 128 * 128;          // 128 rows x 64 bf16 (one SW128 K chunk)
constexpr uint32_t CH_WSTAGE = 64 * 256 * 2;      // 64 K rows x up to 256 N
constexpr int CH_BIAS = kChainMaxL * 256;

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sig_fast(float z) { return fmaf(0.5f, tanh_approx(0.5f * z), 0.5f); }

__device__ __forceinline__ uint32_t ch_sw128(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2);
}

template <int MODE>   // 0 = forward, 1 = backward dX chain
__global__ void __launch_bounds__(384, 1) tc_chain_kernel(const __grid_constant__ ChainMaps maps0,
                                                          const __grid_constant__ ChainMaps maps1,
                                                          const ChainParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAct = smem;
  uint8_t* sW = sAct + CH_ACT_CHUNKS * CH_CHUNK;
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
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % CH_STAGES;
        mbar_wait(&w_empty[s], ((g / CH_STAGES) & 1) ^ 1);
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
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        if (l > 0) mbar_wait(&act_ready[kb], (l - 1) & 1);   // chunk kb of this layer's input
        const int s = g % CH_STAGES;
        mbar_wait(&w_full[s], (g / CH_STAGES) & 1);
        tc_fence_after();
        const uint32_t wb = smem_u32(sW + s * CH_WSTAGE);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = smem_desc_sw128(act_base + kb * CH_CHUNK + ks * 32, 16, 1024);
          const uint64_t bd = MODE == 0 ? smem_desc_sw128(wb + ks * 2048, 8192, 1024)
                                        : smem_desc_sw128(wb + ks * 32, 16, 1024);
          mma_bf16(acc, ad, bd, idesc, (kb | ks) != 0);
        }
        mma_commit(&w_empty[s]);
      }
      mma_commit(&acc_full[l & 1]);
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------------- epilogue (2 warpgroups)
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int row = m0 + r;
    const bool rv = row < p.M;
    if (MODE == 0) {                                   // all biases of this encoder -> SMEM
      for (int l = 0; l < L; ++l)
        for (int c = threadIdx.x - 128; c < E.layer[l].N; c += 256) sBias[l * 256 + c] = E.layer[l].bias[c];
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    float stat = 0.f;
    for (int l = 0; l < L; ++l) {
      const ChainLayer& Ly = E.layer[l];
      const bool last = l == L - 1;
      const int N = Ly.N;
      const int nch = N / 64;
      const uint32_t acc = tmem + (uint32_t)((l & 1) * 256);
      // this warpgroup's column range
      const int cbeg = (nch == 1) ? (wg == 0 ? 0 : N) : (wg == 0 ? 0 : (nch + 1) / 2 * 64);
      const int cend = (nch == 1) ? (wg == 0 ? N : N) : (wg == 0 ? (nch + 1) / 2 * 64 : N);
      uint4 zp[16];                                    // BWD: this half of the Z_{l-1} row
      if (MODE == 1 && rv) {
        const uint4* zr = reinterpret_cast<const uint4*>(Ly.zprev + (size_t)row * N + cbeg);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cbeg + 8 * j < cend) zp[j] = zr[j];
      }
      mbar_wait(&acc_full[l & 1], (l >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < 128; cc += 32) {           // at most 128 columns per warpgroup
        const int c0 = cbeg + cc;
        if (c0 >= cend) break;
        uint32_t raw[32];
        tmem_ld32_nowait(acc + ((uint32_t)(q * 32) << 16) + c0, raw);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
        uint32_t pk[16];                               // bf16 pairs of the value written on
        if (MODE == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += sBias[l * 256 + c0 + i];
          if (!last) {
            uint32_t zk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              zk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
              float a0 = v[2 * i], a1 = v[2 * i + 1];
              a0 = p.act == CRL_ACT_SILU ? a0 * sig_fast(a0) : fmaxf(a0, 0.f);
              a1 = p.act == CRL_ACT_SILU ? a1 * sig_fast(a1) : fmaxf(a1, 0.f);
              pk[i] = pack_bf16x2(a0, a1);
            }
            if (rv) {
              uint4* zo = reinterpret_cast<uint4*>(Ly.out_z + (size_t)row * N + c0);
              uint4* xo = reinterpret_cast<uint4*>(Ly.out_act + (size_t)row * N + c0);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                zo[u] = make_uint4(zk[4 * u], zk[4 * u + 1], zk[4 * u + 2], zk[4 * u + 3]);
                xo[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
              const float2 yb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[i]));
              stat = fmaf(yb.x, yb.x, fmaf(yb.y, yb.y, stat));
            }
            if (rv) {
              float4* yo = reinterpret_cast<float4*>(Ly.out_f + (size_t)row * N + c0);
#pragma unroll
              for (int u = 0; u < 8; ++u) yo[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
              uint4* xo = reinterpret_cast<uint4*>(Ly.out_act + (size_t)row * N + c0);
#pragma unroll
              for (int u = 0; u < 4; ++u) xo[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t zw = reinterpret_cast<const uint32_t*>(zp)[(cc >> 1) + i];
            const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zw));
            float g0, g1;
            if (p.act == CRL_ACT_SILU) {
              const float s0 = sig_fast(z.x), s1 = sig_fast(z.y);
              g0 = s0 * fmaf(z.x, 1.f - s0, 1.f);
              g1 = s1 * fmaf(z.y, 1.f - s1, 1.f);
            } else {
              g0 = z.x > 0.f ? 1.f : 0.f;
              g1 = z.y > 0.f ? 1.f : 0.f;
            }
            pk[i] = pack_bf16x2(v[2 * i] * g0, v[2 * i + 1] * g1);
          }
          if (rv) {
            uint4* o = reinterpret_cast<uint4*>(Ly.out_act + (size_t)row * N + c0);
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
        }
        if (!(MODE == 0 && last)) {
          // next step's A operand: bf16 into the SW128 K-major SMEM chunk (rows >= M write 0s)
          uint8_t* ch = sAct + (c0 >> 6) * CH_CHUNK;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 val = rv ? make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3])
                                 : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(ch + ch_sw128(r, (c0 & 63) + 8 * u)) = val;
          }
          if (((c0 + 32) & 63) == 0 && l + 1 < L) {    // a full 64-feature chunk is written
            tc_fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&act_ready[c0 >> 6]);
          }
        }
      }
    }
    if (MODE == 0) {
      // row statistic of Y: warpgroup 1 hands its columns' partial sum to warpgroup 0
      float* sStat = sBias;                            // biases are no longer needed
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 1) sStat[r] = stat;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 0 && rv && E.out_stat != nullptr) {
        const float st = stat + sStat[r];
        E.out_stat[row] = p.energy == CRL_ENERGY_L2 ? st
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
}

size_t tc_chain_smem() {
  return 1024 + CH_ACT_CHUNKS * CH_CHUNK + CH_STAGES * CH_WSTAGE + CH_BIAS * 4 + 256;
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
  return launch_pdl(tc_chain_kernel<MODE>, grid, dim3(384), smem, st, m0, m1, p);
}

cudaError_t tc_chain_forward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st) {
  return launch_chain<0>(m0, m1, p, 2, st);
}
cudaError_t tc_chain_backward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st) {
  return launch_chain<1>(m0, m1, p, 2, st);
}

}  // namespace tc
}  // namespace crl
