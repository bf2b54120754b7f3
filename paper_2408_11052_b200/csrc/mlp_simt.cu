#include <algorithm>
#include <cstdlib>
// mlp_simt.cu — fp32 SIMT GEMMs for the phi/psi encoders (A2 forward, A5 backward).
//
// Paper: §3.1 P:193-195 (phi(s,a), psi(g)), Table 2, §5.4 (width/depth).
// Layer l: Z = X W + b, X' = act(Z) (hidden) / Y = X W + b (output, reading A-16).
// Backward: dW = X^T dZ, db = colsum(dZ), dX = dZ W^T, dZ_prev = dX * act'(Z_prev).
//
// One templated kernel covers the three GEMM orientations:
//   forward   C[B][out]  = X[B][in]      . W[in][out]     (A row-major,  B row-major)
//   dX        C[B][in]   = dZ[B][out]    . W^T            (A row-major,  B "transposed")
//   dW        C[in][out] = X^T[in][B]    . dZ[B][out]     (A "transposed", B row-major)
// with fused epilogues (bias + activation, activation-derivative, store + column sum for
// db).  The phi input [s || a] is read from two sources without a concat copy (the feature
// index splits at `fsplit`).
//
// Pipeline: 3-stage cp.async (4-byte, zero-filled out of range, so any ld / alignment
// works), BK = 16.  Tiles 64x64 (4x4 per thread) or 32x32 (2x2 per thread) chosen so the
// grid covers the 148 SMs.  The dW GEMMs reduce over the batch: they are split along K
// into S slices written to separate partial buffers (deterministic; summed by the Adam
// kernel or by reduce_partials before an all-reduce).
#include "common.cuh"

namespace crl {

enum GemmEpi { EPI_BIAS_ACT = 0, EPI_BIAS = 1, EPI_DACT = 2, EPI_STORE_COLSUM = 3 };

struct GemmArgs {
  int M, N, K;
  const float* A; int lda;          // primary A source
  const float* A2; int lda2;        // second source for feature index >= fsplit (or null)
  int fsplit;
  const float* B; int ldb;
  float* C; int ldc;                // main output (Z, Y, dZ_prev or dW)
  float* C2;                        // EPI_BIAS_ACT: act(Z) output (ld = ldc)
  const float* bias;                // EPI_BIAS*
  const float* Zp;                  // EPI_DACT: pre-activation of the previous layer (ld = ldc)
  float* colsum;                    // EPI_STORE_COLSUM: db[N] (sum over K of B)
  size_t split_stride;              // floats between K-split partial outputs (C and colsum)
  int k_per_split;
  int act;
};

constexpr int BK = 16, STAGES = 3;

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <bool A_T>
__device__ __forceinline__ const float* a_src(const GemmArgs& p, int m, int k, bool& ok) {
  ok = (m < p.M) && (k < p.K);
  if (!ok) return p.A;
  const int f = A_T ? m : k;                      // feature index
  if (p.A2 != nullptr && f >= p.fsplit)
    return A_T ? p.A2 + (size_t)k * p.lda2 + (m - p.fsplit) : p.A2 + (size_t)m * p.lda2 + (k - p.fsplit);
  return A_T ? p.A + (size_t)k * p.lda + m : p.A + (size_t)m * p.lda + k;
}

template <bool B_T>
__device__ __forceinline__ const float* b_src(const GemmArgs& p, int k, int n, bool& ok) {
  ok = (k < p.K) && (n < p.N);
  if (!ok) return p.B;
  return B_T ? p.B + (size_t)n * p.ldb + k : p.B + (size_t)k * p.ldb + n;
}

template <bool A_T, bool B_T, int EPI, int BM, int BN>
__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgs p) {
  constexpr int TM = BM / 16, TN = BN / 16;       // per-thread micro tile
  constexpr int AP = BM + 4, BP = BN + 4;         // 16-byte aligned rows
  __shared__ __align__(16) float As[STAGES][BK][AP];
  __shared__ __align__(16) float Bs[STAGES][BK][BP];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int split = blockIdx.z;
  const int kbeg = split * p.k_per_split;
  const int kend = min(p.K, kbeg + p.k_per_split);
  const bool do_colsum = (EPI == EPI_STORE_COLSUM) && blockIdx.y == 0;
  pdl_wait();
  pdl_launch();

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  float csum[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) csum[j] = 0.f;

  auto issue = [&](int stage, int k0) {
    constexpr int AE = BM * BK / 256, BE = BN * BK / 256;
#pragma unroll
    for (int r = 0; r < AE; ++r) {
      const int e = tid + r * 256;
      int mm, kk;
      if (!A_T) { mm = e / BK; kk = e % BK; } else { kk = e / BM; mm = e % BM; }
      bool ok;
      const int kg = k0 + kk;
      const float* src = a_src<A_T>(p, m0 + mm, kg < kend ? kg : p.K, ok);
      cp_async4(&As[stage][kk][mm], src, ok);
    }
#pragma unroll
    for (int r = 0; r < BE; ++r) {
      const int e = tid + r * 256;
      int nn, kk;
      if (!B_T) { kk = e / BN; nn = e % BN; } else { nn = e / BK; kk = e % BK; }
      bool ok;
      const int kg = k0 + kk;
      const float* src = b_src<B_T>(p, kg < kend ? kg : p.K, n0 + nn, ok);
      cp_async4(&Bs[stage][kk][nn], src, ok);
    }
  };

  const int ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) issue(s, kbeg + s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) issue(nk % STAGES, kbeg + nk * BK);
      cp_async_commit();
    }
    const int st = kt % STAGES;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
      if (TM == 4) {
        float4 v = *reinterpret_cast<const float4*>(&As[st][kk][ty * 4]);
        a[0] = v.x; a[1] = v.y; a[2 % TM] = v.z; a[3 % TM] = v.w;
      } else {
        float2 v = *reinterpret_cast<const float2*>(&As[st][kk][ty * 2]);
        a[0] = v.x; a[1 % TM] = v.y;
      }
      if (TN == 4) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[st][kk][tx * 4]);
        b[0] = v.x; b[1] = v.y; b[2 % TN] = v.z; b[3 % TN] = v.w;
      } else {
        float2 v = *reinterpret_cast<const float2*>(&Bs[st][kk][tx * 2]);
        b[0] = v.x; b[1 % TN] = v.y;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (do_colsum && ty == 0) {
#pragma unroll
        for (int j = 0; j < TN; ++j) csum[j] += b[j];
      }
    }
  }
  cp_async_wait<0>();

  float* C = p.C + (size_t)split * p.split_stride;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n >= p.N) continue;
      const size_t o = (size_t)m * p.ldc + n;
      float v = acc[i][j];
      if (EPI == EPI_BIAS_ACT) {
        v += p.bias[n];
        C[o] = v;
        p.C2[o] = act_f(v, p.act);
      } else if (EPI == EPI_BIAS) {
        C[o] = v + p.bias[n];
      } else if (EPI == EPI_DACT) {
        C[o] = p.Zp != nullptr ? v * act_grad_f(p.Zp[o], p.act) : v;   // null: plain dX
      } else {
        C[o] = v;
      }
    }
  }
  if (do_colsum && ty == 0) {
    float* cs = p.colsum + (size_t)split * p.split_stride;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < p.N) cs[n] = csum[j];
    }
  }
}

static int g_num_sms = 148;
void gemm_set_num_sms(int n) { g_num_sms = n > 0 ? n : 148; }

template <bool A_T, bool B_T, int EPI>
static cudaError_t launch_gemm(GemmArgs p, int splits, cudaStream_t st) {
  if (splits < 1) splits = 1;
  // every slice s < splits is written (slices past K write zeros), so callers can sum
  // exactly `splits` partial buffers
  p.k_per_split = ((p.K + splits - 1) / splits + BK - 1) / BK * BK;
  const long big = (long)((p.N + 63) / 64) * ((p.M + 63) / 64) * splits;
  if (big >= g_num_sms) {
    dim3 grid((p.N + 63) / 64, (p.M + 63) / 64, splits);
    return launch_pdl(gemm_f32_kernel<A_T, B_T, EPI, 64, 64>, grid, dim3(256), 0, st, p);
  } else {
    dim3 grid((p.N + 31) / 32, (p.M + 31) / 32, splits);
    return launch_pdl(gemm_f32_kernel<A_T, B_T, EPI, 32, 32>, grid, dim3(256), 0, st, p);
  }
  return cudaGetLastError();
}

// Z = X W + b ; Xn = act(Z)     (hidden layer)   or   Y = X W + b   (Xn == nullptr: output)
cudaError_t mlp_forward_layer_f32(int Bn, int in, int out, const float* X, int ldx,
                                  const float* X2, int ldx2, int fsplit, const float* W,
                                  const float* b, float* Z, float* Xn, int act, cudaStream_t st) {
  GemmArgs p{};
  p.M = Bn; p.N = out; p.K = in;
  p.A = X; p.lda = ldx; p.A2 = X2; p.lda2 = ldx2; p.fsplit = fsplit;
  p.B = W; p.ldb = out;
  p.C = Z; p.ldc = out; p.C2 = Xn; p.bias = b; p.act = act;
  if (Xn != nullptr) return launch_gemm<false, false, EPI_BIAS_ACT>(p, 1, st);
  return launch_gemm<false, false, EPI_BIAS>(p, 1, st);
}

// dZ_prev = (dZ W^T) * act'(Z_prev)   (Zprev == nullptr: dX = dZ W^T; W may point at a row
// block of a larger [in_total][out] matrix, e.g. the action rows of the first phi layer)
cudaError_t mlp_backward_dx_f32(int Bn, int in, int out, const float* dZ, const float* W,
                                const float* Zprev, float* dZprev, int act, cudaStream_t st) {
  GemmArgs p{};
  p.M = Bn; p.N = in; p.K = out;
  p.A = dZ; p.lda = out;
  p.B = W; p.ldb = out;                     // B^T[k][n] = W[n][k]
  p.C = dZprev; p.ldc = in; p.Zp = Zprev; p.act = act;
  return launch_gemm<false, true, EPI_DACT>(p, 1, st);
}

// dW[s] = X^T dZ over batch slice s ; db[s] = colsum(dZ) over slice s   (s < splits)
cudaError_t mlp_backward_dw_f32(int Bn, int in, int out, const float* X, int ldx, const float* X2,
                                int ldx2, int fsplit, const float* dZ, float* dW, float* db,
                                int splits, size_t split_stride, cudaStream_t st) {
  GemmArgs p{};
  p.M = in; p.N = out; p.K = Bn;
  p.A = X; p.lda = ldx; p.A2 = X2; p.lda2 = ldx2; p.fsplit = fsplit;
  p.B = dZ; p.ldb = out;
  p.C = dW; p.ldc = out; p.colsum = db; p.split_stride = split_stride;
  return launch_gemm<true, false, EPI_STORE_COLSUM>(p, splits, st);
}

// The number of batch slices the dW GEMMs use for batch Bn (same on every call).
int dw_splits_for(int Bn) {
  if (const char* e = std::getenv("CRL_DW_SPLITS")) return std::max(1, std::min(16, std::atoi(e)));
  int s = Bn / 512;
  return s < 1 ? 1 : (s > 8 ? 8 : s);
}

// g[i] = sum_s part[s * stride + i] for i < n  (in place into slice 0)
__global__ void reduce_partials_kernel(float* part, size_t n, size_t stride, int S) {
  pdl_wait();
  pdl_launch();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float v = part[i];
    for (int s = 1; s < S; ++s) v += part[(size_t)s * stride + i];
    part[i] = v;
  }
}

cudaError_t launch_reduce_partials_range(float* part, size_t n, size_t stride, int S, cudaStream_t st) {
  size_t blocks = (n + 255) / 256;
  if (blocks > (size_t)g_num_sms * 8) blocks = (size_t)g_num_sms * 8;
  if (blocks == 0) blocks = 1;
  return launch_pdl(reduce_partials_kernel, dim3((unsigned)blocks), dim3(256), 0, st, part, n, stride, S);
}

cudaError_t launch_reduce_partials(float* part, size_t n, int S, cudaStream_t st) {
  return launch_reduce_partials_range(part, n, n, S, st);
}

}  // namespace crl
