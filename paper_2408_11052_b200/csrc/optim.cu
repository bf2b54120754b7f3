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
#include "loss_common.cuh"
#include <math_constants.h>

namespace crl {

// Warp per row (coalesced), 64 rows per CTA; every CTA writes its partial sums and the
// last CTA to finish (atomic ticket) adds them in CTA order — deterministic.  acc[0..2] =
// local sums of (LSE_i - l_ii), (LSE'_i - l_ii), LSE_i^2.  If `finalize`, also writes
// loss_out[0..3], sets *skip when the loss is non-finite and advances the Adam step counter.
constexpr int kLossRowsPerCta = 16;    // 2 rows per warp: one DRAM round trip per CTA


__global__ void __launch_bounds__(256) loss_partial_kernel(
    const float* __restrict__ phi, const float* __restrict__ psi, int Bl, int D, int energy,
    const float* __restrict__ lse_row, const float* __restrict__ lse_col, float* __restrict__ acc,
    float* __restrict__ part, unsigned* __restrict__ ticket, int finalize, float invN, float c_f,
    float c_b, float beta, float* __restrict__ loss_out, int* __restrict__ skip,
    int* __restrict__ adam_t, int* __restrict__ status) {
  __shared__ float red[3][8];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float s1 = 0.f, s2 = 0.f, s3 = 0.f;
  const int r0 = blockIdx.x * kLossRowsPerCta;
  pdl_wait();
  pdl_launch();
  for (int q = w; q < kLossRowsPerCta; q += 8) {
    const int i = r0 + q;
    if (i >= Bl) break;
    const float* a = phi + (size_t)i * D;
    const float* b = psi + (size_t)i * D;
    float x = 0.f, na = 0.f, nb = 0.f;
    for (int k = lane; k < D; k += 32) {
      const float av = a[k], bv = b[k];
      if (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_L2SQ) { const float d = av - bv; x = fmaf(d, d, x); }
      else if (energy == CRL_ENERGY_L1) x += fabsf(av - bv);
      else { x = fmaf(av, bv, x); na = fmaf(av, av, na); nb = fmaf(bv, bv, nb); }
    }
    x = warp_sum(x);
    float l;
    if (energy == CRL_ENERGY_L2) l = -sqrtf(x + kEpsL2);
    else if (energy == CRL_ENERGY_L2SQ || energy == CRL_ENERGY_L1) l = -x;
    else if (energy == CRL_ENERGY_DOT) l = x;
    else {
      na = warp_sum(na); nb = warp_sum(nb);
      l = x / (fmaxf(sqrtf(na), kEpsCos) * fmaxf(sqrtf(nb), kEpsCos));
    }
    const float lr = lse_row[i], lc = lse_col[i];
    s1 += lr - l; s2 += lc - l; s3 += lr * lr;
  }
  if (lane == 0) { red[0][w] = s1; red[1][w] = s2; red[2][w] = s3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t1 = 0.f, t2 = 0.f, t3 = 0.f;
    for (int j = 0; j < 8; ++j) { t1 += red[0][j]; t2 += red[1][j]; t3 += red[2][j]; }
    part[blockIdx.x * 4 + 0] = t1; part[blockIdx.x * 4 + 1] = t2; part[blockIdx.x * 4 + 2] = t3;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // last CTA: all 256 threads add the CTA partials (strided, then a fixed-order tree)
  __threadfence();
  __shared__ float tr[3][256];
  float t1 = 0.f, t2 = 0.f, t3 = 0.f;
  for (unsigned j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    t1 += __ldcg(part + j * 4 + 0); t2 += __ldcg(part + j * 4 + 1); t3 += __ldcg(part + j * 4 + 2);
  }
  tr[0][threadIdx.x] = t1; tr[1][threadIdx.x] = t2; tr[2][threadIdx.x] = t3;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h)
      for (int c = 0; c < 3; ++c) tr[c][threadIdx.x] += tr[c][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    acc[0] = tr[0][0]; acc[1] = tr[1][0]; acc[2] = tr[2][0];
    *ticket = 0u;                                  // re-armed for the next (graph) replay
    if (finalize) loss_finalize_dev(acc, invN, c_f, c_b, beta, loss_out, skip, adam_t, status);
  }
}

// Multi-rank: acc[] already all-reduced.
__global__ void loss_finalize_kernel(const float* __restrict__ acc, float invN, float c_f,
                                     float c_b, float beta, float* __restrict__ loss_out,
                                     int* __restrict__ skip, int* __restrict__ adam_t,
                                     int* __restrict__ status) {
  pdl_wait();
  pdl_launch();
  loss_finalize_dev(acc, invN, c_f, c_b, beta, loss_out, skip, adam_t, status);
}

// Fused Adam over the flat fp32 parameters; optional bf16 shadow of the parameters
// (operands of the tensor-core path) written in the same pass.
__global__ void __launch_bounds__(256) adam_kernel(
    float* __restrict__ p, float* __restrict__ g, int S, float* __restrict__ m,
    float* __restrict__ v, size_t n, float lr, float b1, float b2, float eps, float wd,
    const int* __restrict__ adam_t, const int* __restrict__ skip, int* __restrict__ status,
    __nv_bfloat16_raw* __restrict__ shadow, int keep_sum, size_t gs) {
  // gs: floats between the split-K slices of g (the whole gradient's size when this launch
  // updates a sub-range of it)
  pdl_wait();
  pdl_launch();
  if (*skip) return;
  const int t = *adam_t;
  const float bc1 = (float)(1.0 - pow((double)b1, (double)t));
  const float bc2 = (float)(1.0 - pow((double)b2, (double)t));
  const float inv_bc1 = 1.0f / bc1;
  const float inv_sbc2 = 1.0f / sqrtf(bc2);
  bool bad = false;
  // an element whose gradient is not finite is left untouched (p, m, v keep their values; the
  // status word reports CRL_ENONFINITE): a non-finite gradient can never poison the master
  // parameters, the moments or the bf16 shadow (the loss-level check above skips the whole
  // step; this gate covers a finite loss with a non-finite gradient element)
  auto upd = [&](float pi, float gi, float& mi, float& vi) -> float {
    if (!isfinite(gi)) { bad = true; return pi; }
    mi = b1 * mi + (1.f - b1) * gi;
    vi = b2 * vi + (1.f - b2) * gi * gi;
    const float denom = sqrtf(vi) * inv_sbc2 + eps;       // sqrt(v / bc2) + eps
    return pi - lr * ((mi * inv_bc1) / denom + wd * pi);
  };
  const size_t n4 = (n % 4 == 0) ? n / 4 : 0;             // vector path (16-byte accesses)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 gv = reinterpret_cast<const float4*>(g)[i];
    for (int sl = 1; sl < S; ++sl) {                       // deterministic split-K sum
      const float4 h = reinterpret_cast<const float4*>(g + (size_t)sl * gs)[i];
      gv.x += h.x; gv.y += h.y; gv.z += h.z; gv.w += h.w;
    }
    if (S > 1 && keep_sum) reinterpret_cast<float4*>(g)[i] = gv;   // the reduced gradient, for grads_out
    float4 pv = reinterpret_cast<const float4*>(p)[i];
    float4 mv = reinterpret_cast<const float4*>(m)[i];
    float4 vv = reinterpret_cast<const float4*>(v)[i];
    pv.x = upd(pv.x, gv.x, mv.x, vv.x);
    pv.y = upd(pv.y, gv.y, mv.y, vv.y);
    pv.z = upd(pv.z, gv.z, mv.z, vv.z);
    pv.w = upd(pv.w, gv.w, mv.w, vv.w);
    reinterpret_cast<float4*>(p)[i] = pv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (shadow) {
      uint2 hv;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(pv.x, pv.y), h1 = __floats2bfloat162_rn(pv.z, pv.w);
      hv.x = *reinterpret_cast<uint32_t*>(&h0);
      hv.y = *reinterpret_cast<uint32_t*>(&h1);
      reinterpret_cast<uint2*>(shadow)[i] = hv;
    }
  }
  for (size_t i = n4 * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {                // scalar path (n % 4 != 0)
    float gi = g[i];
    for (int sl = 1; sl < S; ++sl) gi += g[(size_t)sl * gs + i];
    if (S > 1) g[i] = gi;
    float mi = m[i], vi = v[i];
    const float pn = upd(p[i], gi, mi, vi);
    m[i] = mi; v[i] = vi; p[i] = pn;
    if (shadow) {
      __nv_bfloat16 h = __float2bfloat16_rn(pn);
      shadow[i] = *reinterpret_cast<__nv_bfloat16_raw*>(&h);
    }
  }
  if (bad) set_status(status, CRL_ENONFINITE);
}

// ---------------------------------------------------------------------------------------
// F3 pair / FB losses (oracle/losses.py pairwise_loss).  d_i = l_ii (warp per row), then one
// CTA adds the per-row sums in a fixed order:
//   L_pair = (1/N) sum_i (Lrow_i + extra_i),  extra = -e^{d_i} (FB), N (d_i - 1)^2 (SPPO)
//   P = beta (1/N) sum_i LSE_i^2,  loss_out = (L_pair, 0, P, L_pair + P)
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pair_diag_kernel(const float* __restrict__ phi, const float* __restrict__ psi,
                                                        int Bl, int D, int energy, float* __restrict__ d) {
  pdl_wait();
  pdl_launch();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= Bl) return;
  const float* a = phi + (size_t)i * D;
  const float* b = psi + (size_t)i * D;
  float x = 0.f, na = 0.f, nb = 0.f;
  for (int k = lane; k < D; k += 32) {
    const float av = a[k], bv = b[k];
    if (energy == CRL_ENERGY_L2 || energy == CRL_ENERGY_L2SQ) { const float t = av - bv; x = fmaf(t, t, x); }
    else if (energy == CRL_ENERGY_L1) x += fabsf(av - bv);
    else { x = fmaf(av, bv, x); na = fmaf(av, av, na); nb = fmaf(bv, bv, nb); }
  }
  x = warp_sum(x);
  float l;
  if (energy == CRL_ENERGY_L2) l = -sqrtf(x + kEpsL2);
  else if (energy == CRL_ENERGY_L2SQ || energy == CRL_ENERGY_L1) l = -x;
  else if (energy == CRL_ENERGY_DOT) l = x;
  else {
    na = warp_sum(na); nb = warp_sum(nb);
    l = x / (fmaxf(sqrtf(na), kEpsCos) * fmaxf(sqrtf(nb), kEpsCos));
  }
  if (lane == 0) d[i] = l;
}

__global__ void __launch_bounds__(1024) pair_loss_kernel(const float* __restrict__ Lrow, const float* __restrict__ d,
                                                         const float* __restrict__ lse, int Bl, int loss, float invN,
                                                         float beta, float* __restrict__ loss_out, float* __restrict__ acc,
                                                         int* __restrict__ skip, int* __restrict__ adam_t,
                                                         int* __restrict__ status) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[2][32];
  float s = 0.f, q = 0.f;
  const float Nf = 1.f / invN;
  for (int i = threadIdx.x; i < Bl; i += blockDim.x) {
    float e = Lrow[i];
    if (loss == CRL_LOSS_FB) e -= expf(d[i]);
    if (loss == CRL_LOSS_SPPO) e += Nf * (d[i] - 1.f) * (d[i] - 1.f);
    s += e;
    q += lse[i] * lse[i];
  }
  s = warp_sum(s);
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s; red[1][threadIdx.x >> 5] = q; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  float a = threadIdx.x < (blockDim.x >> 5) ? red[0][threadIdx.x] : 0.f;
  float b = threadIdx.x < (blockDim.x >> 5) ? red[1][threadIdx.x] : 0.f;
  a = warp_sum(a);
  b = warp_sum(b);
  if (threadIdx.x != 0) return;
  const float L = a * invN, P = beta * b * invN, tot = L + P;
  acc[0] = L; acc[1] = 0.f; acc[2] = P;
  if (loss_out) { loss_out[0] = L; loss_out[1] = 0.f; loss_out[2] = P; loss_out[3] = tot; }
  const bool bad = !isfinite(tot);
  *skip = bad ? 1 : 0;
  if (bad) set_status(status, CRL_ENONFINITE);
  else *adam_t += 1;
}

cudaError_t launch_pair_diag(const float* phi, const float* psi, int Bl, int D, int energy, float* d,
                             cudaStream_t st) {
  return launch_pdl(pair_diag_kernel, dim3((Bl * 32 + 255) / 256), dim3(256), 0, st, phi, psi, Bl, D, energy, d);
}
cudaError_t launch_pair_loss(const float* Lrow, const float* d, const float* lse, int Bl, int loss, float invN,
                             float beta, float* loss_out, float* acc, int* skip, int* adam_t, int* status,
                             cudaStream_t st) {
  return launch_pdl(pair_loss_kernel, dim3(1), dim3(1024), 0, st, Lrow, d, lse, Bl, loss, invN, beta, loss_out, acc,
                    skip, adam_t, status);
}

int loss_partial_blocks(int Bl) { return (Bl + kLossRowsPerCta - 1) / kLossRowsPerCta; }

cudaError_t launch_loss_partial(const float* phi, const float* psi, int Bl, int D, int energy,
                                const float* lse_row, const float* lse_col, float* acc,
                                float* part, unsigned* ticket, int finalize, float invN, float c_f,
                                float c_b, float beta, float* loss_out, int* skip, int* adam_t,
                                int* status, cudaStream_t st) {
  return launch_pdl(loss_partial_kernel, dim3(loss_partial_blocks(Bl)), dim3(256), 0, st, phi, psi, Bl, D,
                    energy, lse_row, lse_col, acc, part, ticket, finalize, invN, c_f, c_b, beta, loss_out,
                    skip, adam_t, status);
}

cudaError_t launch_loss_finalize(const float* acc, float invN, float c_f, float c_b, float beta,
                                 float* loss_out, int* skip, int* adam_t, int* status,
                                 cudaStream_t st) {
  return launch_pdl(loss_finalize_kernel, dim3(1), dim3(1), 0, st, acc, invN, c_f, c_b, beta, loss_out,
                    skip, adam_t, status);
}

cudaError_t launch_adam_ex(float* p, float* g, int S, float* m, float* v, size_t n, float lr,
                           float b1, float b2, float eps, float wd, const int* adam_t,
                           const int* skip, int* status, void* shadow_bf16, int num_sms, int keep_sum,
                           cudaStream_t st);
cudaError_t launch_adam(float* p, float* g, int S, float* m, float* v, size_t n, float lr,
                        float b1, float b2, float eps, float wd, const int* adam_t,
                        const int* skip, int* status, void* shadow_bf16, int num_sms,
                        cudaStream_t st) {
  return launch_adam_ex(p, g, S, m, v, n, lr, b1, b2, eps, wd, adam_t, skip, status, shadow_bf16, num_sms, 1, st);
}

// keep_sum = 0: the split-K partials are summed in registers only (nobody reads the reduced
// gradient after the update: no grads_out), saving one write of the gradient buffer
cudaError_t launch_adam_ex(float* p, float* g, int S, float* m, float* v, size_t n, float lr,
                           float b1, float b2, float eps, float wd, const int* adam_t,
                           const int* skip, int* status, void* shadow_bf16, int num_sms, int keep_sum,
                           cudaStream_t st) {
  size_t blocks = (n / 4 + 255) / 256 + 1;
  size_t cap = (size_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return launch_pdl(adam_kernel, dim3((unsigned)blocks), dim3(256), 0, st, p, g, S, m, v, n, lr, b1, b2, eps,
                    wd, adam_t, skip, status, reinterpret_cast<__nv_bfloat16_raw*>(shadow_bf16), keep_sum, n);
}
// a sub-range [off, off + n) of the parameters whose gradient slices are gs floats apart
cudaError_t launch_adam_range(float* p, float* g, int S, size_t gs, float* m, float* v, size_t n, float lr,
                              float b1, float b2, float eps, float wd, const int* adam_t, const int* skip,
                              int* status, void* shadow_bf16, int num_sms, int keep_sum, cudaStream_t st) {
  size_t blocks = (n / 4 + 255) / 256 + 1;
  size_t cap = (size_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return launch_pdl(adam_kernel, dim3((unsigned)blocks), dim3(256), 0, st, p, g, S, m, v, n, lr, b1, b2, eps,
                    wd, adam_t, skip, status, reinterpret_cast<__nv_bfloat16_raw*>(shadow_bf16), keep_sum, gs);
}

}  // namespace crl
