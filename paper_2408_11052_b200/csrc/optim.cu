// optim.cu — loss reduction (A3 epilogue) and the fused Adam update (A6).
//
// Loss (readings A-02..A-05; App. A.2; Alg. 1):
//   L_fwd = (1/N) sum_i (LSE_i - l_ii),  L_bwd = (1/N) sum_j (LSE'_j - l_jj),
//   P = beta (1/N) sum_i LSE_i^2,  L = c_f L_fwd + c_b L_bwd + P.
// The positives l_ii are recomputed here in difference form from phi_i, psi_i (O(N D)).
// Adam (reading A-15; Alg. 1; Table 2): bias-corrected, eps outside the sqrt,
// decoupled weight decay; step counter t lives in device memory so the step can be replayed
// from a CUDA graph.
#include "common.cuh"
#include <math_constants.h>

namespace crl {

// One CTA, fixed reduction order (deterministic).  Writes acc[0..2] = local sums of
// (LSE_i - l_ii), (LSE'_i - l_ii), LSE_i^2.  If `finalize`, also writes loss_out[0..3],
// sets *skip when the loss is non-finite and advances the Adam step counter.
__global__ void __launch_bounds__(1024) loss_partial_kernel(
    const float* __restrict__ phi, const float* __restrict__ psi, int Bl, int D, int energy,
    const float* __restrict__ lse_row, const float* __restrict__ lse_col, float* __restrict__ acc,
    int finalize, float invN, float c_f, float c_b, float beta, float* __restrict__ loss_out,
    int* __restrict__ skip, int* __restrict__ adam_t, int* __restrict__ status) {
  __shared__ float red[3][32];
  float s1 = 0.f, s2 = 0.f, s3 = 0.f;
  for (int i = threadIdx.x; i < Bl; i += blockDim.x) {
    const float* a = phi + (size_t)i * D;
    const float* b = psi + (size_t)i * D;
    float l;
    if (energy == CRL_ENERGY_L2) {
      float d2 = 0.f;
      for (int k = 0; k < D; ++k) { float d = a[k] - b[k]; d2 = fmaf(d, d, d2); }
      l = -sqrtf(d2 + kEpsL2);
    } else {
      float dot = 0.f, na = 0.f, nb = 0.f;
      for (int k = 0; k < D; ++k) { dot = fmaf(a[k], b[k], dot); na = fmaf(a[k], a[k], na); nb = fmaf(b[k], b[k], nb); }
      l = (energy == CRL_ENERGY_DOT) ? dot
                                     : dot / (fmaxf(sqrtf(na), kEpsCos) * fmaxf(sqrtf(nb), kEpsCos));
    }
    const float lr = lse_row[i], lc = lse_col[i];
    s1 += lr - l;
    s2 += lc - l;
    s3 += lr * lr;
  }
  s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[0][w] = s1; red[1][w] = s2; red[2][w] = s3; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s1 = lane < nw ? red[0][lane] : 0.f;
    s2 = lane < nw ? red[1][lane] : 0.f;
    s3 = lane < nw ? red[2][lane] : 0.f;
    s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
    if (lane == 0) {
      acc[0] = s1; acc[1] = s2; acc[2] = s3;
      if (finalize) {
        const float Lf = s1 * invN, Lb = s2 * invN, P = beta * s3 * invN;
        const float tot = c_f * Lf + c_b * Lb + P;
        if (loss_out) { loss_out[0] = Lf; loss_out[1] = Lb; loss_out[2] = P; loss_out[3] = tot; }
        const bool bad = !isfinite(tot);
        *skip = bad ? 1 : 0;
        if (bad) set_status(status, CRL_ENONFINITE);
        else *adam_t += 1;
      }
    }
  }
}

// Multi-rank: acc[] already all-reduced.
__global__ void loss_finalize_kernel(const float* __restrict__ acc, float invN, float c_f,
                                     float c_b, float beta, float* __restrict__ loss_out,
                                     int* __restrict__ skip, int* __restrict__ adam_t,
                                     int* __restrict__ status) {
  const float Lf = acc[0] * invN, Lb = acc[1] * invN, P = beta * acc[2] * invN;
  const float tot = c_f * Lf + c_b * Lb + P;
  if (loss_out) { loss_out[0] = Lf; loss_out[1] = Lb; loss_out[2] = P; loss_out[3] = tot; }
  const bool bad = !isfinite(tot);
  *skip = bad ? 1 : 0;
  if (bad) set_status(status, CRL_ENONFINITE);
  else *adam_t += 1;
}

// Fused Adam over the flat fp32 parameters; optional bf16 shadow of the parameters
// (operands of the tensor-core path) written in the same pass.
__global__ void __launch_bounds__(256) adam_kernel(
    float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
    float* __restrict__ v, size_t n, float lr, float b1, float b2, float eps, float wd,
    const int* __restrict__ adam_t, const int* __restrict__ skip, int* __restrict__ status,
    __nv_bfloat16_raw* __restrict__ shadow) {
  if (*skip) return;
  const int t = *adam_t;
  const float bc1 = (float)(1.0 - pow((double)b1, (double)t));
  const float bc2 = (float)(1.0 - pow((double)b2, (double)t));
  const float inv_bc1 = 1.0f / bc1;
  const float inv_sbc2 = 1.0f / sqrtf(bc2);
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    bad |= !isfinite(gi);
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi; v[i] = vi;
    const float mh = mi * inv_bc1;
    const float denom = sqrtf(vi) * inv_sbc2 + eps;       // sqrt(v / bc2) + eps
    const float pi = p[i];
    const float pn = pi - lr * (mh / denom + wd * pi);
    p[i] = pn;
    if (shadow) {
      __nv_bfloat16 h = __float2bfloat16_rn(pn);
      shadow[i] = *reinterpret_cast<__nv_bfloat16_raw*>(&h);
    }
  }
  if (bad) set_status(status, CRL_ENONFINITE);
}

cudaError_t launch_loss_partial(const float* phi, const float* psi, int Bl, int D, int energy,
                                const float* lse_row, const float* lse_col, float* acc,
                                int finalize, float invN, float c_f, float c_b, float beta,
                                float* loss_out, int* skip, int* adam_t, int* status,
                                cudaStream_t st) {
  loss_partial_kernel<<<1, 1024, 0, st>>>(phi, psi, Bl, D, energy, lse_row, lse_col, acc,
                                          finalize, invN, c_f, c_b, beta, loss_out, skip, adam_t,
                                          status);
  return cudaGetLastError();
}

cudaError_t launch_loss_finalize(const float* acc, float invN, float c_f, float c_b, float beta,
                                 float* loss_out, int* skip, int* adam_t, int* status,
                                 cudaStream_t st) {
  loss_finalize_kernel<<<1, 1, 0, st>>>(acc, invN, c_f, c_b, beta, loss_out, skip, adam_t, status);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, size_t n, float lr,
                        float b1, float b2, float eps, float wd, const int* adam_t,
                        const int* skip, int* status, void* shadow_bf16, int num_sms,
                        cudaStream_t st) {
  size_t blocks = (n + 255) / 256;
  size_t cap = (size_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  adam_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, wd, adam_t, skip,
                                                status,
                                                reinterpret_cast<__nv_bfloat16_raw*>(shadow_bf16));
  return cudaGetLastError();
}

}  // namespace crl
