// tc_gradf.h — host interface of the fused two-sided gradient pass (tc_gradf.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace crl {
namespace tc {

// The loss reduction folded into the gradient kernel (its idle warps); part == nullptr: the
// caller computes the loss elsewhere.
struct GradfLoss {
  const float* phi32 = nullptr;   // [N][64] fp32 representations (the positives l_ii)
  const float* psi32 = nullptr;
  float* part = nullptr;          // [row blocks][4] scratch
  unsigned* ticket = nullptr;     // zero on entry, re-armed by the kernel
  float* acc = nullptr;           // [3] sums (LSE_i - l_ii), (LSE'_i - l_ii), LSE_i^2
  float* out = nullptr;           // [4] L_fwd, L_bwd, penalty, total (or null)
  int* skip = nullptr;            // Adam skip flag (non-finite loss)
  int* adam_t = nullptr;          // Adam step counter (advanced when finite)
  int* status = nullptr;
  float c_f = 1.f, c_b = 1.f, beta = 0.f;
};

// one side of the two-call online-max statistics (tc_logits.cu tc_logits_lse_pair)
struct LseSide {
  const CUtensorMap* mA; const CUtensorMap* mB;
  const float* a_stat; const float* b_stat;
  float* part_m; float* part_s;     // [S][Na] split partials
  float* lse; float* fac;           // [Na] outputs
  float cc0, cc1;                   // column-coefficient constants (lse_merge_kernel)
};
cudaError_t tc_logits_lse_pair(int D, int energy, const LseSide& c0, const LseSide& c1, int Na, int Nb, int S,
                               int* fac_ok, int* ticket, const int* gate, cudaStream_t st);

bool tc_gradf_supports(int D, int energy);
int tc_gradf_splits(int Na, int Nb, int num_sms);
bool tc_gradf_map(CUtensorMap* m, float* db_acc, int Nb);
cudaError_t tc_grad_fused(int energy, const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mDB, int Na,
                          int Nb, const float* a_stat, const float* b_stat, const float* lse_row, const float* lse_col,
                          const float* fac_col, const int* fac_ok, float c_r, float c_c, float beta_r, float invN,
                          int S, float* part_da, float* part_rs, float* db_acc, float* cs_acc,
                          const __nv_bfloat16* A, const __nv_bfloat16* B, float* dA, __nv_bfloat16* dAb, float* dB,
                          __nv_bfloat16* dBb, const GradfLoss& loss, cudaStream_t st);

}  // namespace tc
}  // namespace crl
