// ln.cu — LayerNorm before the hidden activations (§5.4 P:462-465 "adding
// layer normalization before every activation", App. A.4), fp32 path.
//
// Reading A-35: per row over the layer's features, learnable gain gamma and shift beta,
// eps = 1e-6 inside the square root.  Per hidden layer (oracle/mlp.py forward_ln):
//   Zh = (Z - mu) rstd,  rstd = 1 / sqrt(var + eps),  Y = gamma Zh + beta,  X' = act(Y)
// backward, with dY = dX' act'(Y) (the dX GEMM epilogue evaluates act' at Y):
//   dZ = rstd (g - mean(g) - Zh mean(g Zh)),  g = gamma dY
//   dgamma = sum_rows dY Zh,  dbeta = sum_rows dY
// One warp per row for the row reductions.  The parameter gradients follow the split-K
// convention of the dW kernels: split s (a contiguous row range) writes slice s, one CTA per
// split, warps added in a fixed order (deterministic; Adam sums the slices).
#include "common.cuh"

namespace crl {

constexpr float kLnEps = 1e-6f;

__global__ void __launch_bounds__(256) ln_fwd_kernel(int Bn, int N, const float* __restrict__ Z,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     int act, float* __restrict__ Y, float* __restrict__ Xn,
                                                     float* __restrict__ mu, float* __restrict__ rstd) {
  pdl_wait();
  pdl_launch();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= Bn) return;
  const float* z = Z + (size_t)row * N;
  float s = 0.f;
  for (int k = lane; k < N; k += 32) s += z[k];
  const float m = warp_sum(s) / (float)N;
  float v = 0.f;
  for (int k = lane; k < N; k += 32) { const float d = z[k] - m; v = fmaf(d, d, v); }
  const float r = rsqrtf(warp_sum(v) / (float)N + kLnEps);
  for (int k = lane; k < N; k += 32) {
    const float y = fmaf(gamma[k], (z[k] - m) * r, beta[k]);
    Y[(size_t)row * N + k] = y;
    Xn[(size_t)row * N + k] = act == CRL_ACT_SILU ? y / (1.f + __expf(-y)) : fmaxf(y, 0.f);
  }
  if (lane == 0) { mu[row] = m; rstd[row] = r; }
}

// dY -> dZ in place; dgamma / dbeta slices.  grid = splits, 256 threads.
__global__ void __launch_bounds__(256) ln_bwd_kernel(int Bn, int N, float* __restrict__ dYZ,
                                                      const float* __restrict__ Z, const float* __restrict__ mu,
                                                      const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                      float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                      int rows_per_split, size_t split_stride) {
  extern __shared__ float sacc[];                        // [2][N]
  pdl_wait();
  pdl_launch();
  const int split = blockIdx.x;
  const int r0 = split * rows_per_split, r1 = min(Bn, r0 + rows_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) sacc[k] = 0.f;
  constexpr int kMaxPer = 64;                            // N <= 2048
  float ag[kMaxPer], ab[kMaxPer];
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) { ag[u] = 0.f; ab[u] = 0.f; }
  for (int row = r0 + warp; row < r1; row += nw) {
    float* dy = dYZ + (size_t)row * N;
    const float* z = Z + (size_t)row * N;
    const float m = mu[row], r = rstd[row];
    float sg = 0.f, sgz = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPer; ++u) {
      const int k = lane + 32 * u;
      if (k < N) {
        const float zh = (z[k] - m) * r;
        const float d = dy[k];
        const float g = gamma[k] * d;
        sg += g; sgz = fmaf(g, zh, sgz);
        ag[u] = fmaf(d, zh, ag[u]);
        ab[u] += d;
      }
    }
    const float mg = warp_sum(sg) / (float)N, mgz = warp_sum(sgz) / (float)N;
#pragma unroll
    for (int u = 0; u < kMaxPer; ++u) {
      const int k = lane + 32 * u;
      if (k < N) {
        const float zh = (z[k] - m) * r;
        const float g = gamma[k] * dy[k];
        dy[k] = r * (g - mg - zh * mgz);
      }
    }
  }
  __syncthreads();
  for (int w = 0; w < nw; ++w) {                         // fixed warp order: deterministic
    if (warp == w) {
#pragma unroll
      for (int u = 0; u < kMaxPer; ++u) {
        const int k = lane + 32 * u;
        if (k < N) { sacc[k] += ag[u]; sacc[N + k] += ab[u]; }
      }
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    dgamma[(size_t)split * split_stride + k] = sacc[k];
    dbeta[(size_t)split * split_stride + k] = sacc[N + k];
  }
}

cudaError_t launch_ln_fwd(int Bn, int N, const float* Z, const float* gamma, const float* beta, int act, float* Y,
                          float* Xn, float* mu, float* rstd, cudaStream_t st) {
  return launch_pdl(ln_fwd_kernel, dim3((Bn * 32 + 255) / 256), dim3(256), 0, st, Bn, N, Z, gamma, beta, act, Y,
                    Xn, mu, rstd);
}

cudaError_t launch_ln_bwd(int Bn, int N, float* dYZ, const float* Z, const float* mu, const float* rstd,
                          const float* gamma, float* dgamma, float* dbeta, int splits, size_t split_stride,
                          cudaStream_t st) {
  if (N > 2048) return cudaErrorInvalidValue;
  const int rps = (Bn + splits - 1) / splits;
  const size_t smem = (size_t)2 * N * sizeof(float);
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ln_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(ln_bwd_kernel, dim3(splits), dim3(256), smem, st, Bn, N, dYZ, Z, mu, rstd, gamma, dgamma,
                    dbeta, rps, split_stride);
}

}  // namespace crl
