// loss_common.cuh — the loss finalisation shared by the loss kernels (optim.cu) and the
// loss-reducing gradient merge (tc_logits.cu).  Readings A-02..A-05, A-24 (FlatNCE).
#pragma once
#include "common.cuh"

namespace crl {

// acc[0..2] = sum_i (LSE_i - l_ii), sum_i (LSE'_i - l_ii), sum_i LSE_i^2 over the global batch
__device__ __forceinline__ void loss_finalize_dev(const float* acc, float invN, float c_f,
                                                  float c_b, float beta, float* loss_out,
                                                  int* skip, int* adam_t, int* status) {
  // negative coefficients mark the FlatNCE losses (F3, reading A-24): same InfoNCE sums and
  // gradient, but the reported value of log(S / sg[S]) is 0 (the finiteness test keeps the sums)
  const bool flat = c_f < 0.f || c_b < 0.f;
  c_f = fabsf(c_f); c_b = fabsf(c_b);
  const float Lf = acc[0] * invN, Lb = acc[1] * invN, P = beta * acc[2] * invN;
  const float tot = c_f * Lf + c_b * Lb + P;
  if (loss_out) {
    loss_out[0] = flat ? 0.f : Lf; loss_out[1] = flat ? 0.f : Lb; loss_out[2] = P;
    loss_out[3] = flat ? P : tot;
  }
  const bool bad = !isfinite(tot);
  *skip = bad ? 1 : 0;
  if (bad) {
    set_status(status, CRL_ENONFINITE);
  } else {
    *adam_t += 1;
  }
}

}  // namespace crl
