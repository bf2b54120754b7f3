// tc_dwg.cu — every weight and bias gradient of both encoders in ONE launch (A5, BF16 path).
//
// Paper: backward of the encoders of §3.1 P:193-195 (Alg. 1 P:1051 "gradient"):
//   dW_l = X_l^T dZ_l  (M = in, N = out, K = batch)      db_l = 1^T dZ_l  (column sums)
// A grouped tcgen05 GEMM: blockIdx.x enumerates (problem, K split, M block, N block) tiles of
// up to 16 problems (2 encoders x <= 8 layers); each problem carries its own TMA maps (X_l and
// dZ_l as stored, both MN-major operands: no transposed copies).  The bias gradient rides on
// the same SMEM dZ tiles: CTAs of M block 0 issue a second MMA per K step with an all-ones A
// operand, so TMEM columns [256, 256 + bn) accumulate 1^T dZ (every row equal) next to dW.
// Tiles are 128 x bn with bn = the full output width up to 256 (one N block per layer at
// width 256): each X^T tile is read once per M block, which halves the L2 -> SM traffic of
// 128 x 64 tiles (the GEMM is operand-bandwidth bound: K = batch is long, M, N are small).
// Split-K slices are written to deterministic partial buffers (summed by Adam), as before.
// Replaces 2 launches per layer (tc_gemm dW + colsum) with one for the whole backward.
#include "common.cuh"
#include "tc_common.cuh"
#include <cstdlib>

#include "tc_dwg.h"

namespace crl {
namespace tc {

namespace {
constexpr int GM = 128, GNMAX = 256, GK = 64, GST = 4;
constexpr uint32_t GA_BYTES = GM * GK * 2;        // 16 KB: X^T tile (two 64-row MN chunks)
constexpr uint32_t GB_BYTES = GNMAX * GK * 2;     // 32 KB: dZ tile (up to 256 columns)
constexpr uint32_t GONES_BYTES = GM * GK * 2;     // 16 KB all-ones A operand
constexpr size_t kDwgSmem = 1024 + GST * (GA_BYTES + GB_BYTES) + GONES_BYTES + 256;
}  // namespace

__global__ void __launch_bounds__(256, 1) tc_dwg_kernel(const __grid_constant__ DwgParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + GST * GA_BYTES;
  uint8_t* sOnes = sB + GST * GB_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + GONES_BYTES);
  uint64_t* empty = full + GST;
  uint64_t* tfull = empty + GST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  // ---- which tile of which problem
  int t = blockIdx.x, pi = 0;
  while (pi + 1 < P.n && t >= P.prob[pi].tiles) { t -= P.prob[pi].tiles; ++pi; }
  const DwgProblem& pr = P.prob[pi];
  const int nb = pr.nblk, mb = pr.mblk;
  const int split = t / (mb * nb);
  const int rem = t % (mb * nb);
  const int mbi = rem / nb, nbi = rem % nb;
  const int bn = pr.bn;                            // 64..256 columns per tile (runtime MMA N)
  const int m0 = mbi * GM, n0 = nbi * bn;
  const int kbeg = split * P.k_per_split;
  const int kend = min(P.K, kbeg + P.k_per_split);
  const int nkb = kend > kbeg ? (kend - kbeg + GK - 1) / GK : 0;
  const bool do_db = mbi == 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&pr.mapX);
    tma_prefetch_desc(&pr.mapDZ);
    for (int s = 0; s < GST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);       // dW: [0, bn), 1^T dZ: [256, 256 + bn)
  if (do_db) {
    for (int i = threadIdx.x; i < (int)(GONES_BYTES / 16); i += blockDim.x)
      reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch();

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % GST;
      mbar_wait(&empty[s], ((kb / GST) & 1) ^ 1);
      mbar_expect_tx(&full[s], GA_BYTES + (uint32_t)bn * GK * 2);
      const int k = kbeg + kb * GK;
      uint8_t* a_dst = sA + s * GA_BYTES;
#pragma unroll
      for (int c = 0; c < GM / 64; ++c) tma_load_2d(a_dst + c * GK * 128, &pr.mapX, &full[s], m0 + 64 * c, k);
      for (int c = 0; c < bn / 64; ++c) tma_load_2d(sB + s * GB_BYTES + c * GK * 128, &pr.mapDZ, &full[s], n0 + 64 * c, k);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(GM, bn, true, true);
    const uint32_t idesc1 = idesc_bf16_f32(GM, bn, false, true);      // ones (any layout) . dZ
    const uint32_t ones = smem_u32(sOnes);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % GST;
      mbar_wait(&full[s], (kb / GST) & 1);
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA + s * GA_BYTES);
      const uint32_t b_base = smem_u32(sB + s * GB_BYTES);
#pragma unroll
      for (int ks = 0; ks < GK / 16; ++ks) {
        const uint64_t bd = smem_desc_sw128(b_base + ks * 2048, GK * 128, 1024);
        mma_bf16(tmem, smem_desc_sw128(a_base + ks * 2048, GK * 128, 1024), bd, idesc, (kb | ks) != 0);
        if (do_db) mma_bf16(tmem + 256, smem_desc_sw128(ones + ks * 32, 16, 1024), bd, idesc1, (kb | ks) != 0);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tfull);
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 4;
    const int row = m0 + q * 32 + lane;
    const bool rv = row < pr.M;
    mbar_wait(tfull, 0);
    tc_fence_after();
    float* dw = pr.dW + (size_t)split * P.split_stride;
    if (pr.tma_w) {
      // TMEM -> SW128 fp32 staging in the (now idle) B stages: bn / 32 boxes of 128 rows x 32
      // columns, 16 KB each -> TMA stores (whole 128 B row segments instead of per-thread
      // 16 B pieces of 1 KB-strided rows)
      const int r = q * 32 + lane;
      const uint32_t stg = smem_u32(sB) + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
#pragma unroll 1
      for (int c0 = 0; c0 < bn; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        if (nkb == 0) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        const uint32_t cb = stg + (uint32_t)(c0 >> 5) * 16384u;
        const int g0 = (c0 & 31) >> 2;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(cb + (uint32_t)(((g0 + i) ^ (r & 7)) << 4)),
                       "f"(v[4 * i]), "f"(v[4 * i + 1]), "f"(v[4 * i + 2]), "f"(v[4 * i + 3])
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        for (int j = 0; j < bn / 32; ++j)
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&pr.mapW)),
                       "r"(smem_u32(sB) + (uint32_t)j * 16384u), "r"(n0 + 32 * j), "r"(m0), "r"(split)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
#pragma unroll 1
    for (int c0 = 0; c0 < bn; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
      if (nkb == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      const int n = n0 + c0;
      const int nvalid = min(16, pr.N - n);
      if (rv && nvalid > 0) {
        float* dst = dw + (size_t)row * pr.N + n;
        if (nvalid >= 16) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          for (int i = 0; i < nvalid; ++i) dst[i] = v[i];
        }
      }
    }
    }
    if (do_db && q == 0) {
      // every TMEM row of the second accumulator holds the 64 column sums of this tile
      float* db = pr.db + (size_t)split * P.split_stride;
#pragma unroll 1
      for (int c0 = 0; c0 < bn; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + 256 + c0, v);
        float mine = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) mine = (i == (lane & 15)) ? v[i] : mine;
        if (nkb == 0) mine = 0.f;
        const int n = n0 + c0 + lane;
        if (lane < 16 && n < pr.N) db[n] = mine;
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

bool make_map_bf16(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
bool make_map_f32_3d(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);

bool dwg_add_problem(DwgParams& P, const __nv_bfloat16* X, int ldx, const __nv_bfloat16* dZ, int M, int N,
                     float* dW, float* db) {
  if (P.n >= kDwgMaxProblems) return false;
  DwgProblem& pr = P.prob[P.n];
  // X [K = batch][ldx] read as the MN-major A operand (M = in features, 64-wide boxes);
  // dZ [K][N] as the MN-major B operand
  if (!make_map_bf16(&pr.mapX, X, M, P.K, ldx, 64, 64) || !make_map_bf16(&pr.mapDZ, dZ, N, P.K, N, 64, 64))
    return false;
  pr.M = M; pr.N = N; pr.dW = dW; pr.db = db;
  // TMA-store epilogue when the partial slices are 16 B aligned (rows: N, slices: split_stride)
  pr.tma_w = !std::getenv("CRL_DWG_NO_TMA_STORE") && (reinterpret_cast<uintptr_t>(dW) % 16 == 0) &&
             (N % 4 == 0) && (P.split_stride % 4 == 0) &&
             make_map_f32_3d(&pr.mapW, dW, N, M, P.splits, N, P.split_stride, 32, 128);
  // wide tiles only pay once K (= batch) is long; short K is latency bound: more, narrower
  // tiles spread the epilogue over more SMs (measured: B = 256 prefers 64, B >= 4096 256)
  pr.bn = P.K < 2048 ? 64 : (N >= GNMAX ? GNMAX : (N + 63) / 64 * 64);
  pr.mblk = (M + GM - 1) / GM;
  pr.nblk = (N + pr.bn - 1) / pr.bn;
  pr.tiles = pr.mblk * pr.nblk * P.splits;
  P.total_tiles += pr.tiles;
  ++P.n;
  return true;
}

void dwg_init(DwgParams& P, int K, int splits, size_t split_stride) {
  P = DwgParams{};
  P.K = K;
  P.splits = splits;
  P.k_per_split = ((K + splits - 1) / splits + GK - 1) / GK * GK;
  P.split_stride = split_stride;
}

cudaError_t tc_dwg_launch(const DwgParams& P, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_dwg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDwgSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (P.total_tiles == 0) return cudaSuccess;
  return launch_pdl(tc_dwg_kernel, dim3(P.total_tiles), dim3(256), kDwgSmem, st, P);
}

}  // namespace tc
}  // namespace crl
