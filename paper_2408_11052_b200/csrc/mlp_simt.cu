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
// with fused epilogues (bias + activation, activation-derivative, plain store + column sum
// for db).  The phi input [s || a] is read from two sources without a concat copy (the
// feature index splits at `fsplit`).  64x64 tile, BK = 16, 256 threads, 4x4 per thread.
#include "common.cuh"

namespace crl {

enum GemmEpi { EPI_BIAS_ACT = 0, EPI_BIAS = 1, EPI_DACT = 2, EPI_STORE_COLSUM = 3, EPI_STORE = 4 };

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
  int act;
};

constexpr int BM = 64, BN = 64, BK = 16;

template <bool A_T, bool B_T>
__device__ __forceinline__ float load_a(const GemmArgs& p, int m, int k) {
  // feature index: k for A row-major (X[m][k]); m for A transposed (X^T[m][k] = X[k][m])
  if (m >= p.M || k >= p.K) return 0.0f;
  if (!A_T) {
    if (p.A2 != nullptr && k >= p.fsplit) return p.A2[(size_t)m * p.lda2 + (k - p.fsplit)];
    return p.A[(size_t)m * p.lda + k];
  } else {
    if (p.A2 != nullptr && m >= p.fsplit) return p.A2[(size_t)k * p.lda2 + (m - p.fsplit)];
    return p.A[(size_t)k * p.lda + m];
  }
}

template <bool B_T>
__device__ __forceinline__ float load_b(const GemmArgs& p, int k, int n) {
  if (k >= p.K || n >= p.N) return 0.0f;
  return B_T ? p.B[(size_t)n * p.ldb + k] : p.B[(size_t)k * p.ldb + n];
}

template <bool A_T, bool B_T, int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgs p) {
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const bool do_colsum = (EPI == EPI_STORE_COLSUM) && blockIdx.y == 0;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  float csum[4] = {0.f, 0.f, 0.f, 0.f};

  // each thread loads 4 A and 4 B elements per K-tile
  auto load_tiles = [&](int buf, int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + r * 256;           // 0..1023 over a 64x16 tile
      if (!A_T) {                      // coalesce along k: e -> (m = e / 16, k = e % 16)
        int mm = e >> 4, kk = e & 15;
        As[buf][kk][mm] = load_a<A_T, B_T>(p, m0 + mm, k0 + kk);
      } else {                         // coalesce along m: e -> (k = e / 64, m = e % 64)
        int kk = e >> 6, mm = e & 63;
        As[buf][kk][mm] = load_a<A_T, B_T>(p, m0 + mm, k0 + kk);
      }
      if (!B_T) {                      // coalesce along n
        int kk = e >> 6, nn = e & 63;
        Bs[buf][kk][nn] = load_b<B_T>(p, k0 + kk, n0 + nn);
      } else {                         // coalesce along k
        int nn = e >> 4, kk = e & 15;
        Bs[buf][kk][nn] = load_b<B_T>(p, k0 + kk, n0 + nn);
      }
    }
  };

  const int ktiles = (p.K + BK - 1) / BK;
  load_tiles(0, 0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tiles(buf ^ 1, (kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 av = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      float4 bv = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      float a[4] = {av.x, av.y, av.z, av.w};
      float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (do_colsum && ty == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) csum[j] += b[j];
      }
    }
    __syncthreads();
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= p.N) continue;
      const size_t o = (size_t)m * p.ldc + n;
      float v = acc[i][j];
      if (EPI == EPI_BIAS_ACT) {
        v += p.bias[n];
        p.C[o] = v;
        p.C2[o] = act_f(v, p.act);
      } else if (EPI == EPI_BIAS) {
        p.C[o] = v + p.bias[n];
      } else if (EPI == EPI_DACT) {
        p.C[o] = v * act_grad_f(p.Zp[o], p.act);
      } else {
        p.C[o] = v;
      }
    }
  }
  if (do_colsum && ty == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < p.N) p.colsum[n] = csum[j];
    }
  }
}

template <bool A_T, bool B_T, int EPI>
static cudaError_t launch_gemm(const GemmArgs& p, cudaStream_t st) {
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM);
  gemm_f32_kernel<A_T, B_T, EPI><<<grid, 256, 0, st>>>(p);
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
  if (Xn != nullptr) return launch_gemm<false, false, EPI_BIAS_ACT>(p, st);
  return launch_gemm<false, false, EPI_BIAS>(p, st);
}

// dZ_prev = (dZ W^T) * act'(Z_prev)
cudaError_t mlp_backward_dx_f32(int Bn, int in, int out, const float* dZ, const float* W,
                                const float* Zprev, float* dZprev, int act, cudaStream_t st) {
  GemmArgs p{};
  p.M = Bn; p.N = in; p.K = out;
  p.A = dZ; p.lda = out;
  p.B = W; p.ldb = out;                     // B^T[k][n] = W[n][k]
  p.C = dZprev; p.ldc = in; p.Zp = Zprev; p.act = act;
  return launch_gemm<false, true, EPI_DACT>(p, st);
}

// dW = X^T dZ ; db = colsum(dZ)
cudaError_t mlp_backward_dw_f32(int Bn, int in, int out, const float* X, int ldx, const float* X2,
                                int ldx2, int fsplit, const float* dZ, float* dW, float* db,
                                cudaStream_t st) {
  GemmArgs p{};
  p.M = in; p.N = out; p.K = Bn;
  p.A = X; p.lda = ldx; p.A2 = X2; p.lda2 = ldx2; p.fsplit = fsplit;
  p.B = dZ; p.ldb = out;
  p.C = dW; p.ldc = out; p.colsum = db;
  return launch_gemm<true, false, EPI_STORE_COLSUM>(p, st);
}

}  // namespace crl
