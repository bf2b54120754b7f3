// tc_gemm.cu — bf16 tcgen05 GEMMs (TMA -> SMEM -> tcgen05.mma -> TMEM -> epilogue) for the
// phi/psi encoders on the BF16 path (A2 forward, A5 backward).
//
// Paper: §3.1 P:193-195 (phi(s,a), psi(g)), Table 2, §5.4 P:387-465.
//   forward  Z[B][out]  = X[B][in]  . W[in][out]   A K-major,   B MN-major (W as stored)
//   dX       dX[B][in]  = dZ[B][out] . W^T          A K-major,   B K-major  (W as stored)
//   dW       dW[in][out] = X^T . dZ (K = batch)     A MN-major,  B MN-major (X, dZ as stored)
// so no transposed copies are ever made: the operand major-ness is a descriptor bit.
//
// Kernel anatomy (one 128 x BN output tile per CTA, 256 threads):
//   warp 0 / lane 0 : TMA producer, STAGES-deep ring of (A, B) K-blocks of 64 (SW128)
//   warp 1 / lane 0 : tcgen05.mma issuer (M=128, N=BN, K=16 per instruction), commits each
//                     stage back to the producer and the accumulator to the epilogue
//   warp 2          : TMEM allocation (BN fp32 columns)
//   warps 4..7      : epilogue, one TMEM lane (= output row) per thread, tcgen05.ld x16,
//                     fused bias / activation / activation-derivative, vector stores
// Split-K along blockIdx.z writes deterministic fp32 partial slices (dW).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"

namespace crl {
namespace tc {

enum TcEpi { TEPI_FWD_HIDDEN = 0, TEPI_FWD_OUT = 1, TEPI_DX = 2, TEPI_DW = 3 };

struct TcGemmArgs {
  int M, N, K, k_per_split;
  const float* bias;               // FWD_*: [N] fp32 master bias
  __nv_bfloat16* out_bf;           // FWD_HIDDEN: act(Z); FWD_OUT: Y; DX: dZ_prev
  __nv_bfloat16* out_z;            // FWD_HIDDEN: Z (bf16)
  int ld_bf;                       // pitch (elements) of out_bf / out_z / zprev
  float* out_f;                    // FWD_OUT: Y fp32; DW: dW partial slices
  int ld_f;
  size_t split_stride;             // floats between DW partial slices
  const __nv_bfloat16* zprev;      // DX: pre-activation of the previous layer
  int act;
  float* out_stat;                 // FWD_OUT (single N tile): row statistic of bf16(Y) for the
  int stat_energy;                 //   logits stage (L2: |y|^2, cos: 1/max(|y|, eps)), else null
  int trace;                       // measurement: globaltimer phases of CTA 0 (CRL_GEMM_TRACE)
};

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int BM = 128, BK = 64, STAGES = 4;

template <int BN>
struct TcSmem {
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr size_t bytes = 1024 + STAGES * (A_BYTES + B_BYTES) + 256 + BN * 4;
};

__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float (&v)[16], int nvalid) {
  if (nvalid >= 16) {
    uint4 a, b;
    a.x = pack_bf16x2(v[0], v[1]);   a.y = pack_bf16x2(v[2], v[3]);
    a.z = pack_bf16x2(v[4], v[5]);   a.w = pack_bf16x2(v[6], v[7]);
    b.x = pack_bf16x2(v[8], v[9]);   b.y = pack_bf16x2(v[10], v[11]);
    b.z = pack_bf16x2(v[12], v[13]); b.w = pack_bf16x2(v[14], v[15]);
    reinterpret_cast<uint4*>(dst)[0] = a;
    reinterpret_cast<uint4*>(dst)[1] = b;
  } else {
    for (int i = 0; i < nvalid; ++i) dst[i] = __float2bfloat16_rn(v[i]);
  }
}
__device__ __forceinline__ void store_f32x16(float* dst, const float (&v)[16], int nvalid) {
  if (nvalid >= 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
    for (int i = 0; i < nvalid; ++i) dst[i] = v[i];
  }
}
__device__ __forceinline__ void load_bf16x16(const __nv_bfloat16* src, float (&v)[16], int nvalid) {
  if (nvalid >= 16) {
    uint4 a = reinterpret_cast<const uint4*>(src)[0], b = reinterpret_cast<const uint4*>(src)[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      float2 f = __bfloat1622float2(h);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
    }
  } else {
    for (int i = 0; i < 16; ++i) v[i] = i < nvalid ? __bfloat162float(src[i]) : 0.f;
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(256, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         TcGemmArgs p) {
  using S = TcSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * S::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);   // followed by sbias[BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * p.k_per_split;
  const int kend = min(p.K, kbeg + p.k_per_split);
  const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const bool trace = p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  __shared__ unsigned long long s_tt[8];
  if (trace && threadIdx.x == 0) s_tt[0] = gtimer();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // prologue above (barriers, TMEM, descriptor prefetch) overlaps the predecessor's tail; the
  // weight operand (FWD / DX: B = W, written by the previous step's Adam) does not depend on
  // the predecessor either, so its first STAGES K-blocks are requested before the wait
  constexpr bool B_IS_W = EPI != TEPI_DW;
  const int npre = B_IS_W ? min(nkb, STAGES) : 0;
  auto load_b = [&](int kb, int s) {
    const int k = kbeg + kb * BK;
    uint8_t* b_dst = sB + s * S::B_BYTES;
    if (!B_MN) {
      tma_load_2d(b_dst, &tmB, &full[s], k, n0);                    // dims {K, N}
    } else {
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tma_load_2d(b_dst + c * BK * 128, &tmB, &full[s], n0 + 64 * c, k);
    }
  };
  if (trace && threadIdx.x == 0) s_tt[1] = gtimer();
  if (warp == 0 && lane == 0)
    for (int kb = 0; kb < npre; ++kb) {
      mbar_expect_tx(&full[kb], S::A_BYTES + S::B_BYTES);
      load_b(kb, kb);
    }
  pdl_wait();
  pdl_launch();
  if (trace && threadIdx.x == 0) s_tt[2] = gtimer();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      if (kb >= npre) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], S::A_BYTES + S::B_BYTES);
        load_b(kb, s);
      }
      const int k = kbeg + kb * BK;
      uint8_t* a_dst = sA + s * S::A_BYTES;
      if (!A_MN) {
        tma_load_2d(a_dst, &tmA, &full[s], k, m0);                  // dims {K, M}
      } else {
#pragma unroll
        for (int c = 0; c < BM / 64; ++c) tma_load_2d(a_dst + c * BK * 128, &tmA, &full[s], m0 + 64 * c, k);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      if (trace && kb == 0) s_tt[3] = gtimer();
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA + s * S::A_BYTES);
      const uint32_t b_base = smem_u32(sB + s * S::B_BYTES);
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        const uint64_t ad = A_MN ? smem_desc_sw128(a_base + ks * 2048, BK * 128, 1024)
                                 : smem_desc_sw128(a_base + ks * 32, 16, 1024);
        const uint64_t bd = B_MN ? smem_desc_sw128(b_base + ks * 2048, BK * 128, 1024)
                                 : smem_desc_sw128(b_base + ks * 32, 16, 1024);
        mma_bf16(tmem, ad, bd, idesc, (kb | ks) != 0);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tfull);
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 4;
    const int row = m0 + q * 32 + lane;
    const bool rv = row < p.M;
    // operands of the epilogue are fetched while the mainloop runs (one DRAM round trip,
    // not one per 16-column chunk)
    float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
    if (EPI == TEPI_FWD_HIDDEN || EPI == TEPI_FWD_OUT) {
      for (int c = threadIdx.x - 128; c < BN; c += 128) sbias[c] = (n0 + c < p.N) ? p.bias[n0 + c] : 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    uint4 zp[EPI == TEPI_DX ? BN / 8 : 1];
    if (EPI == TEPI_DX && rv) {
      const __nv_bfloat16* zrow = p.zprev + (size_t)row * p.ld_bf + n0;
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) {
        if (n0 + 8 * j + 8 <= p.N) {
          zp[j] = reinterpret_cast<const uint4*>(zrow)[j];
        } else {
          __nv_bfloat16 t[8];
          for (int i = 0; i < 8; ++i) t[i] = (n0 + 8 * j + i < p.N) ? zrow[8 * j + i] : __float2bfloat16_rn(0.f);
          zp[j] = *reinterpret_cast<uint4*>(t);
        }
      }
    }
    mbar_wait(tfull, 0);
    if (trace && threadIdx.x == 128) s_tt[4] = gtimer();
    tc_fence_after();
    float ysq = 0.f;                                     // FWD_OUT: sum of bf16(y)^2 of the row
    // the whole BN-column row in one burst of TMEM loads (one wait), then branch-free math:
    // the activation is a kernel-uniform choice hoisted out of the per-element code, and SiLU /
    // SiLU' use tanh.approx (sigma(z) = (1 + tanh(z/2)) / 2: one MUFU op, no division); the
    // outputs are rounded to bf16 (2^-9), the tanh.approx error is ~2^-11
    uint32_t acc[BN];
#pragma unroll
    for (int c = 0; c < BN / 32; ++c)
      tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(acc + 32 * c));
    tmem_ld_wait();
    if (nkb == 0) {
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0u;
    }
    auto epilogue = [&](auto silu_c) {
      constexpr bool SILU = decltype(silu_c)::value;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(acc[c0 + i]);
        const int n = n0 + c0;
        const int nvalid = min(16, p.N - n);
        if (!rv || nvalid <= 0) continue;
        if (EPI == TEPI_FWD_HIDDEN || EPI == TEPI_FWD_OUT) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sbias[c0 + i];
          if (EPI == TEPI_FWD_HIDDEN) {
            store_bf16x16(p.out_z + (size_t)row * p.ld_bf + n, v, nvalid);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (SILU) {
                const float h = 0.5f * v[i];
                v[i] = fmaf(h, tanh_fast(h), h);
              } else {
                v[i] = fmaxf(v[i], 0.f);
              }
            }
            store_bf16x16(p.out_bf + (size_t)row * p.ld_bf + n, v, nvalid);
          } else {
            store_f32x16(p.out_f + (size_t)row * p.ld_f + n, v, nvalid);
            if (p.out_stat != nullptr) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float yb = __bfloat162float(__float2bfloat16_rn(v[i]));
                ysq = i < nvalid ? fmaf(yb, yb, ysq) : ysq;
              }
            }
            store_bf16x16(p.out_bf + (size_t)row * p.ld_bf + n, v, nvalid);
          }
        } else if (EPI == TEPI_DX) {
          const uint32_t w[8] = {zp[c0 / 8].x, zp[c0 / 8].y, zp[c0 / 8].z, zp[c0 / 8].w,
                                 zp[c0 / 8 + 1].x, zp[c0 / 8 + 1].y, zp[c0 / 8 + 1].z, zp[c0 / 8 + 1].w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
            if (SILU) {
              // silu'(z) = 1/2 + (t + h (1 - t^2)) / 2, h = z/2, t = tanh(h)
              const float h0 = 0.5f * z.x, h1 = 0.5f * z.y;
              const float t0 = tanh_fast(h0), t1 = tanh_fast(h1);
              v[2 * i] *= fmaf(0.5f, fmaf(h0, fmaf(-t0, t0, 1.f), t0), 0.5f);
              v[2 * i + 1] *= fmaf(0.5f, fmaf(h1, fmaf(-t1, t1, 1.f), t1), 0.5f);
            } else {
              v[2 * i] = z.x > 0.f ? v[2 * i] : 0.f;
              v[2 * i + 1] = z.y > 0.f ? v[2 * i + 1] : 0.f;
            }
          }
          store_bf16x16(p.out_bf + (size_t)row * p.ld_bf + n, v, nvalid);
        } else {
          store_f32x16(p.out_f + (size_t)blockIdx.z * p.split_stride + (size_t)row * p.ld_f + n, v, nvalid);
        }
      }
    };
    if (p.act == CRL_ACT_SILU) epilogue(std::true_type{});
    else epilogue(std::false_type{});
    // FWD_OUT with the whole output row in this CTA: the logits stage's row statistic
    // (replaces a separate row-statistic launch; same bf16-rounded vector it will read)
    if (EPI == TEPI_FWD_OUT && p.out_stat != nullptr && rv)
      p.out_stat[row] = (p.stat_energy == CRL_ENERGY_L2 || p.stat_energy == CRL_ENERGY_L2SQ) ? ysq
                        : (p.stat_energy == CRL_ENERGY_COS ? 1.f / fmaxf(sqrtf(ysq), kEpsCos) : 0.f);
    if (trace && threadIdx.x == 128) s_tt[5] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, BN);
  }
  if (trace && threadIdx.x == 0)
    printf("GEMM_TRACE epi=%d M=%d N=%d K=%d grid=%d,%d,%d entry=%llu prologue=%llu pdl=%llu mma0=%llu acc=%llu end=%llu\n",
           EPI, p.M, p.N, p.K, gridDim.x, gridDim.y, gridDim.z, s_tt[0] % 100000000ull, s_tt[1] - s_tt[0],
           s_tt[2] - s_tt[0], s_tt[3] - s_tt[0], s_tt[4] - s_tt[0], s_tt[5] - s_tt[0]);
}

// -------------------------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2-D bf16 tensor map, SWIZZLE_128B, dims {inner, outer}, row pitch in elements.
bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
                   uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D fp32 tensor map, SWIZZLE_128B (box_inner * 4 must be <= 128 B), dims {inner, outer}.
bool make_map_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
                  uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// fp32 [depth][outer][inner] with explicit pitches (elements), SW128 boxes {box_inner, box_outer, 1}
bool make_map_f32_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t depth,
                     uint64_t pitch_elems, uint64_t depth_pitch_elems, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {inner, outer, depth};
  cuuint64_t strides[2] = {pitch_elems * 4, depth_pitch_elems * 4};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, const TcGemmArgs& p, int splits,
                             cudaStream_t st) {
  static bool attr = false;
  const size_t smem = TcSmem<BN>::bytes;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, A_MN, B_MN, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, splits);
  static const int trace = std::getenv("CRL_GEMM_TRACE") ? 1 : 0;
  TcGemmArgs q = p;
  q.trace = trace;
  return launch_pdl(tc_gemm_kernel<BN, A_MN, B_MN, EPI>, grid, dim3(256), smem, st, a, b, q);
}

// Operand maps for one GEMM: boxes follow the kernel's TMA calls.
//   A K-major: {K, M} box {64, 128};  A MN-major: {M, K} box {64, 64}
//   B K-major: {K, N} box {64, BN};   B MN-major: {N, K} box {64, 64}
int tc_pick_bn(int M, int N, int num_sms) {
  if (N <= 64) return 64;
  const long tiles128 = (long)((M + 127) / 128) * ((N + 127) / 128);
  if (tiles128 * 2 <= num_sms) return 64;
  return 128;
}

template <int EPI, bool A_MN, bool B_MN>
static cudaError_t dispatch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const TcGemmArgs& p,
                               int splits, cudaStream_t st) {
  switch (bn) {
    case 64: return launch_tc<64, A_MN, B_MN, EPI>(a, b, p, splits, st);
    case 128: return launch_tc<128, A_MN, B_MN, EPI>(a, b, p, splits, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t tc_forward(int bn, const CUtensorMap& mapX, const CUtensorMap& mapW, int Bn, int in, int out,
                       const float* bias, __nv_bfloat16* z, __nv_bfloat16* xn, int ld_bf, float* y_f32,
                       int ld_f, int act, float* y_stat, int energy, cudaStream_t st) {
  TcGemmArgs p{};
  p.M = Bn; p.N = out; p.K = in; p.k_per_split = in;
  p.bias = bias; p.out_z = z; p.out_bf = xn; p.ld_bf = ld_bf; p.out_f = y_f32; p.ld_f = ld_f; p.act = act;
  p.out_stat = (y_stat != nullptr && out <= bn) ? y_stat : nullptr;     // whole row in one CTA only
  p.stat_energy = energy;
  if (y_f32 == nullptr) return dispatch_bn<TEPI_FWD_HIDDEN, false, true>(bn, mapX, mapW, p, 1, st);
  return dispatch_bn<TEPI_FWD_OUT, false, true>(bn, mapX, mapW, p, 1, st);
}

cudaError_t tc_backward_dx(int bn, const CUtensorMap& mapDZ, const CUtensorMap& mapWk, int Bn, int in, int out,
                           const __nv_bfloat16* zprev, __nv_bfloat16* dzprev, int ld_bf, int act,
                           cudaStream_t st) {
  TcGemmArgs p{};
  p.M = Bn; p.N = in; p.K = out; p.k_per_split = out;
  p.zprev = zprev; p.out_bf = dzprev; p.ld_bf = ld_bf; p.act = act;
  return dispatch_bn<TEPI_DX, false, false>(bn, mapDZ, mapWk, p, 1, st);
}

cudaError_t tc_backward_dw(int bn, const CUtensorMap& mapX_mn, const CUtensorMap& mapDZ_mn, int Bn, int in,
                           int out, float* dW, int splits, size_t split_stride, cudaStream_t st) {
  TcGemmArgs p{};
  p.M = in; p.N = out; p.K = Bn;
  p.k_per_split = ((Bn + splits - 1) / splits + BK - 1) / BK * BK;
  p.out_f = dW; p.ld_f = out; p.split_stride = split_stride;
  return dispatch_bn<TEPI_DW, true, true>(bn, mapX_mn, mapDZ_mn, p, splits, st);
}

// ---------------------------------------------------------------- small helpers (bf16 path)
// X0 for phi: [s || a] -> bf16 [B][ld] (columns >= obs+act are left as written at init = 0);
// X0 for psi: g -> bf16 [B][ldg]
__global__ void prep_inputs_kernel(const float* __restrict__ s, const float* __restrict__ a,
                                   const float* __restrict__ g, int Bn, int obs, int act, int goal,
                                   __nv_bfloat16* __restrict__ x0, int ld0, __nv_bfloat16* __restrict__ g0,
                                   int ldg, int* __restrict__ reset, int* __restrict__ fac_ok, int fac_init,
                                   float* __restrict__ zero, size_t zero_n) {
  const int in0 = obs + act;
  const size_t tot0 = (size_t)Bn * in0, totg = (size_t)Bn * goal;
  pdl_wait();
  pdl_launch();
  if (blockIdx.x == 0 && threadIdx.x == 0) {           // per-step device flags
    if (reset != nullptr) *reset = 0;
    if (fac_ok != nullptr) *fac_ok = fac_init;
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot0 + totg;
       i += (size_t)gridDim.x * blockDim.x) {
    if (i < tot0) {
      const int r = (int)(i / in0), c = (int)(i % in0);
      const float v = c < obs ? s[(size_t)r * obs + c] : a[(size_t)r * act + (c - obs)];
      x0[(size_t)r * ld0 + c] = __float2bfloat16_rn(v);
    } else {
      const size_t j = i - tot0;
      const int r = (int)(j / goal), c = (int)(j % goal);
      g0[(size_t)r * ldg + c] = __float2bfloat16_rn(g[j]);
    }
  }
  // the fused gradient pass's reduction accumulator (a memset node here would cut the
  // programmatic-launch chain of the step graph)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < zero_n; i += (size_t)gridDim.x * blockDim.x)
    zero[i] = 0.f;
}

cudaError_t launch_prep_inputs(const float* s, const float* a, const float* g, int Bn, int obs, int act,
                               int goal, __nv_bfloat16* x0, int ld0, __nv_bfloat16* g0, int ldg,
                               int num_sms, int* reset, int* fac_ok, int fac_init, float* zero, size_t zero_n,
                               cudaStream_t st) {
  size_t tot = (size_t)Bn * (obs + act + goal);
  size_t blocks = (tot + 255) / 256;
  if (blocks > (size_t)num_sms * 4) blocks = (size_t)num_sms * 4;
  return launch_pdl(prep_inputs_kernel, dim3((unsigned)blocks), dim3(256), 0, st, s, a, g, Bn, obs, act, goal,
                    x0, ld0, g0, ldg, reset, fac_ok, fac_init, zero, zero_n);
}

// db[s][n] = sum over the batch slice s of dZ[b][n] (bf16 in, fp32 out): 64 columns x one
// slice per CTA; thread (tx, ty) sums column pair 2tx of rows ty, ty+8, ... with 8 loads in
// flight, then the 8 row phases are added in a fixed order (deterministic).  Same slicing as
// the dW GEMM so Adam can sum the partial slices.
__global__ void __launch_bounds__(256) colsum_bf16_kernel(const __nv_bfloat16* __restrict__ dz, int Bn, int N,
                                                          int ld, float* __restrict__ db, int rows_per_split,
                                                          size_t split_stride) {
  __shared__ float red[8][65];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = blockIdx.x * 64 + 2 * tx;
  const int sl = blockIdx.y;
  const int r0 = sl * rows_per_split, r1 = min(Bn, r0 + rows_per_split);
  float a0 = 0.f, a1 = 0.f;
  pdl_wait();
  pdl_launch();
  if (n < N) {
    const bool pair = n + 1 < N;
    int r = r0 + ty;
    for (; r + 56 < r1; r += 64) {
      float2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat16* p = dz + (size_t)(r + 8 * u) * ld + n;
        v[u] = pair ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p))
                    : make_float2(__bfloat162float(*p), 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { a0 += v[u].x; a1 += v[u].y; }
    }
    for (; r < r1; r += 8) {
      const __nv_bfloat16* p = dz + (size_t)r * ld + n;
      a0 += __bfloat162float(p[0]);
      if (pair) a1 += __bfloat162float(p[1]);
    }
  }
  red[ty][2 * tx] = a0;
  red[ty][2 * tx + 1] = a1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = blockIdx.x * 64 + threadIdx.x;
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += red[j][threadIdx.x];
    if (c < N) db[(size_t)sl * split_stride + c] = t;
  }
}

cudaError_t launch_colsum_bf16(const __nv_bfloat16* dz, int Bn, int N, int ld, float* db, int splits,
                               size_t split_stride, cudaStream_t st) {
  const int rps = ((Bn + splits - 1) / splits + BK - 1) / BK * BK;
  dim3 grid((N + 63) / 64, splits);
  return launch_pdl(colsum_bf16_kernel, grid, dim3(256), 0, st, dz, Bn, N, ld, db, rps, split_stride);
}

// fp32 -> bf16 copy (dPhi / dPsi from the logits kernels feed the output-layer backward)
__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, size_t n) {
  pdl_wait();
  pdl_launch();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}
cudaError_t launch_f32_to_bf16(const float* x, __nv_bfloat16* y, size_t n, int num_sms, cudaStream_t st) {
  size_t blocks = (n + 255) / 256;
  if (blocks > (size_t)num_sms * 4) blocks = (size_t)num_sms * 4;
  return launch_pdl(f32_to_bf16_kernel, dim3((unsigned)blocks), dim3(256), 0, st, x, y, n);
}

}  // namespace tc
}  // namespace crl
