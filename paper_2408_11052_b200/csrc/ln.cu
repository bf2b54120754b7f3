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

// ==================================================================================== bf16
// The BF16 tensor-core path (F2 at width 1,024: the CTA-pair GEMM writes Z = X W + b in bf16,
// these kernels apply the LayerNorm; the dX GEMM's epilogue evaluates act' at Y, these kernels
// turn dY into dZ).  Same maths and reading A-35 as above; bf16 activations, fp32 statistics,
// fp32 parameter gradients.  A warp per row, lane l owns elements [8 l + 256 j, + 8) (16 B
// vector accesses), N = 256 NV.
namespace crl {

template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_bf16_kernel(int Bn, const __nv_bfloat16* __restrict__ Z,
                                                          const float* __restrict__ gamma,
                                                          const float* __restrict__ beta, int act,
                                                          __nv_bfloat16* __restrict__ Y, __nv_bfloat16* __restrict__ Xn,
                                                          float* __restrict__ mu, float* __restrict__ rstd) {
  constexpr int N = 256 * NV;
  pdl_wait();
  pdl_launch();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= Bn) return;
  float z[NV][8];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(Z + (size_t)row * N + 256 * j + 8 * lane);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
      z[j][2 * h] = f.x; z[j][2 * h + 1] = f.y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += z[j][i];
  const float m = warp_sum(s) * (1.f / (float)N);
  float v = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) { const float d = z[j][i] - m; v = fmaf(d, d, v); }
  const float r = rsqrtf(warp_sum(v) * (1.f / (float)N) + kLnEps);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int k0 = 256 * j + 8 * lane;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + k0)), g1 = __ldg(reinterpret_cast<const float4*>(gamma + k0 + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + k0)), b1 = __ldg(reinterpret_cast<const float4*>(beta + k0 + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float y[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      y[i] = fmaf(gg[i], (z[j][i] - m) * r, bb[i]);
      if (act == CRL_ACT_SILU) {                         // SiLU(y) = h + h tanh(h), h = y / 2 (as the GEMM epilogues)
        const float h = 0.5f * y[i];
        float t;
        asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
        x[i] = fmaf(h, t, h);
      } else {
        x[i] = fmaxf(y[i], 0.f);
      }
    }
    uint4 oy, ox;
    __nv_bfloat162 t;
    t = __floats2bfloat162_rn(y[0], y[1]); oy.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(y[2], y[3]); oy.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(y[4], y[5]); oy.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(y[6], y[7]); oy.w = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(x[0], x[1]); ox.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(x[2], x[3]); ox.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(x[4], x[5]); ox.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(x[6], x[7]); ox.w = *reinterpret_cast<uint32_t*>(&t);
    *reinterpret_cast<uint4*>(Y + (size_t)row * N + k0) = oy;
    *reinterpret_cast<uint4*>(Xn + (size_t)row * N + k0) = ox;
  }
  if (lane == 0) { mu[row] = m; rstd[row] = r; }
}

// dY -> dZ in place (bf16); the dgamma / dbeta column sums of this CTA's rows -> part[blk][2N]
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_bf16_kernel(int Bn, int rows_per_blk, __nv_bfloat16* __restrict__ dYZ,
                                                          const __nv_bfloat16* __restrict__ Z,
                                                          const float* __restrict__ mu, const float* __restrict__ rstd,
                                                          const float* __restrict__ gamma, float* __restrict__ part) {
  constexpr int N = 256 * NV;
  __shared__ float red[2 * N];
  pdl_wait();
  pdl_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r0 = blockIdx.x * rows_per_blk, r1 = min(Bn, r0 + rows_per_blk);
  float ag[NV][8], ab[NV][8], gm[NV][8];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + 256 * j + 8 * lane));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + 256 * j + 8 * lane + 4));
    gm[j][0] = g0.x; gm[j][1] = g0.y; gm[j][2] = g0.z; gm[j][3] = g0.w;
    gm[j][4] = g1.x; gm[j][5] = g1.y; gm[j][6] = g1.z; gm[j][7] = g1.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) { ag[j][i] = 0.f; ab[j][i] = 0.f; }
  }
  for (int row = r0 + warp; row < r1; row += nw) {
    const float m = mu[row], r = rstd[row];
    float d[NV][8], zh[NV][8];
    float sg = 0.f, sgz = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const size_t o = (size_t)row * N + 256 * j + 8 * lane;
      const uint4 ud = *reinterpret_cast<const uint4*>(dYZ + o);
      const uint4 uz = *reinterpret_cast<const uint4*>(Z + o);
      const uint32_t wd[4] = {ud.x, ud.y, ud.z, ud.w}, wz[4] = {uz.x, uz.y, uz.z, uz.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float2 fd = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wd[h]));
        const float2 fz = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wz[h]));
        d[j][2 * h] = fd.x; d[j][2 * h + 1] = fd.y;
        zh[j][2 * h] = (fz.x - m) * r; zh[j][2 * h + 1] = (fz.y - m) * r;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float g = gm[j][i] * d[j][i];
        sg += g;
        sgz = fmaf(g, zh[j][i], sgz);
        ag[j][i] = fmaf(d[j][i], zh[j][i], ag[j][i]);
        ab[j][i] += d[j][i];
      }
    }
    const float mg = warp_sum(sg) * (1.f / (float)N), mgz = warp_sum(sgz) * (1.f / (float)N);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = r * (gm[j][i] * d[j][i] - mg - zh[j][i] * mgz);
      uint4 u;
      __nv_bfloat162 t;
      t = __floats2bfloat162_rn(o[0], o[1]); u.x = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(o[2], o[3]); u.y = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(o[4], o[5]); u.z = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(o[6], o[7]); u.w = *reinterpret_cast<uint32_t*>(&t);
      *reinterpret_cast<uint4*>(dYZ + (size_t)row * N + 256 * j + 8 * lane) = u;
    }
  }
  // column sums of the CTA: warps added in a fixed order (deterministic)
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) red[k] = 0.f;
  __syncthreads();
  for (int w = 0; w < nw; ++w) {
    if (warp == w) {
#pragma unroll
      for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          red[256 * j + 8 * lane + i] += ag[j][i];
          red[N + 256 * j + 8 * lane + i] += ab[j][i];
        }
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) part[(size_t)blockIdx.x * 2 * N + k] = red[k];
}

// dgamma / dbeta = the sum of the CTA partials, into K slice 0 of the gradient buffer; the other
// slices (summed by Adam) get zeros.  One CTA per 32 columns: warp w sums partials w, w + 8, ...
// of its lane's column (coalesced 128 B rows, many loads in flight), then the 8 warp sums are
// added in warp order (deterministic).  (One thread per column walking all nblk partials left
// 8 CTAs on the whole GPU: ~30 us per call, latency-bound.)
__global__ void __launch_bounds__(256) ln_param_reduce_kernel(int N, int nblk, const float* __restrict__ part,
                                                              float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                              int S, size_t split_stride) {
  __shared__ float red[8][32];
  pdl_wait();
  pdl_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 32 + lane;
  float t = 0.f;
  if (k < 2 * N) {
    float t1 = 0.f, t2 = 0.f, t3 = 0.f;
    int b = warp;
    for (; b + 24 < nblk; b += 32) {
      t += part[(size_t)b * 2 * N + k];
      t1 += part[(size_t)(b + 8) * 2 * N + k];
      t2 += part[(size_t)(b + 16) * 2 * N + k];
      t3 += part[(size_t)(b + 24) * 2 * N + k];
    }
    for (; b < nblk; b += 8) t += part[(size_t)b * 2 * N + k];
    t = (t + t1) + (t2 + t3);
  }
  red[warp][lane] = t;
  __syncthreads();
  if (warp != 0 || k >= 2 * N) return;
  float o = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) o += red[w][lane];
  float* dst = k < N ? dgamma + k : dbeta + (k - N);
  dst[0] = o;
  for (int s2 = 1; s2 < S; ++s2) dst[(size_t)s2 * split_stride] = 0.f;
}

bool ln_bf16_supports(int N) { return N % 256 == 0 && N >= 256 && N <= 1024; }

cudaError_t launch_ln_fwd_bf16(int Bn, int N, const __nv_bfloat16* Z, const float* gamma, const float* beta, int act,
                               __nv_bfloat16* Y, __nv_bfloat16* Xn, float* mu, float* rstd, cudaStream_t st) {
  const dim3 grid((Bn * 32 + 255) / 256), blk(256);
  switch (N / 256) {
    case 1: return launch_pdl(ln_fwd_bf16_kernel<1>, grid, blk, 0, st, Bn, Z, gamma, beta, act, Y, Xn, mu, rstd);
    case 2: return launch_pdl(ln_fwd_bf16_kernel<2>, grid, blk, 0, st, Bn, Z, gamma, beta, act, Y, Xn, mu, rstd);
    case 3: return launch_pdl(ln_fwd_bf16_kernel<3>, grid, blk, 0, st, Bn, Z, gamma, beta, act, Y, Xn, mu, rstd);
    case 4: return launch_pdl(ln_fwd_bf16_kernel<4>, grid, blk, 0, st, Bn, Z, gamma, beta, act, Y, Xn, mu, rstd);
  }
  return cudaErrorInvalidValue;
}

// part: [nblk][2N] fp32 scratch; nblk CTAs of 256 threads over the rows
cudaError_t launch_ln_bwd_bf16(int Bn, int N, __nv_bfloat16* dYZ, const __nv_bfloat16* Z, const float* mu,
                               const float* rstd, const float* gamma, float* part, int nblk, float* dgamma,
                               float* dbeta, int S, size_t split_stride, cudaStream_t st) {
  const int rpb = (Bn + nblk - 1) / nblk;
  const dim3 grid(nblk), blk(256);
  cudaError_t e = cudaErrorInvalidValue;
  switch (N / 256) {
    case 1: e = launch_pdl(ln_bwd_bf16_kernel<1>, grid, blk, 0, st, Bn, rpb, dYZ, Z, mu, rstd, gamma, part); break;
    case 2: e = launch_pdl(ln_bwd_bf16_kernel<2>, grid, blk, 0, st, Bn, rpb, dYZ, Z, mu, rstd, gamma, part); break;
    case 3: e = launch_pdl(ln_bwd_bf16_kernel<3>, grid, blk, 0, st, Bn, rpb, dYZ, Z, mu, rstd, gamma, part); break;
    case 4: e = launch_pdl(ln_bwd_bf16_kernel<4>, grid, blk, 0, st, Bn, rpb, dYZ, Z, mu, rstd, gamma, part); break;
  }
  if (e != cudaSuccess) return e;
  return launch_pdl(ln_param_reduce_kernel, dim3((2 * N + 31) / 32), dim3(256), 0, st, N, nblk,
                    (const float*)part, dgamma, dbeta, S, split_stride);
}

}  // namespace crl
