// tc_merge.cuh — the per-row merge of split gradient partials (shared by the two-call logits
// kernels, tc_logits.cu, and the fused gradient pass, tc_gradf.cu).
//
// dA[i] = sum_s part[s][i]  (+ energy finalisation), fp32 and bf16 outputs.  One warp per row.
// Also adds the positive-pair (delta_ii) term of dL/dl, -C delta_ij with C = invN (c_r + c_c),
// which the tile epilogues leave out: its energy chain uses the pair (A_i, B_{row_offset+i})
// (L2: 1/r_ii from the difference form; cos: 1/|B_i|).  Readings A-02..A-06.
#pragma once
#include "common.cuh"

#include <cuda_bf16.h>

namespace crl {
namespace tc {

struct GradMergeArgs {
  const float* part; const float* prs; const __nv_bfloat16* A; const float* a_stat;
  const __nv_bfloat16* Bg; const float* b_stat; int row_offset; float Cdiag; int Na, D, S;
  float* out; __nv_bfloat16* outb;
  int pre;   // cos: part already carries the row's own 1/|A_i| (fused pass, w' = g r_i s_j)
  const unsigned char* valid1 = nullptr;   // tc_grad2: slot 1 holds data only for cut row blocks
  int prs_sub = 1;                         // row-sum sub-partials per slot (tc_grad2: 2 warpgroups)
};

template <int ENERGY>
__device__ __forceinline__ void grad_merge_row(const GradMergeArgs& g, int w, int lane) {
  const float* __restrict__ part = g.part;
  const float* __restrict__ prs = g.prs;
  const __nv_bfloat16* __restrict__ A = g.A;
  const float* __restrict__ a_stat = g.a_stat;
  const __nv_bfloat16* __restrict__ Bg = g.Bg;
  const float* __restrict__ b_stat = g.b_stat;
  const int row_offset = g.row_offset, Na = g.Na, D = g.D, S = g.S;
  const float Cdiag = g.Cdiag;
  float* __restrict__ out = g.out;
  __nv_bfloat16* __restrict__ outb = g.outb;
  if (w >= Na) return;
  const size_t ib = (size_t)(row_offset + w) * D;
  // slots that hold data for this row (tc_grad2: the second slot only for cut row blocks)
  const int Sr = (g.valid1 != nullptr && S > 1 && !g.valid1[w >> 7]) ? 1 : S;
  float rs = 0.f;
  if (ENERGY == CRL_ENERGY_L2)
    for (int s = 0; s < Sr * g.prs_sub; ++s) rs += prs[(size_t)s * Na + w];
  float av[8], bv[8], acc[8];                            // D <= 256 -> 8 per lane
  float d2 = 0.f;
  for (int c = 0; c < D / 32; ++c) {
    const int k = lane + 32 * c;
    av[c] = __bfloat162float(A[(size_t)w * D + k]);
    bv[c] = __bfloat162float(Bg[ib + k]);
    const float d = av[c] - bv[c];
    d2 = fmaf(d, d, d2);
  }
  float diag = 0.f;                                      // energy-chain weight of the delta term
  if (ENERGY == CRL_ENERGY_L2) diag = Cdiag / sqrtf(warp_sum(d2) + kEpsL2);   // times (A_i - B_i)
  const float invb = ENERGY == CRL_ENERGY_COS ? b_stat[row_offset + w] : 0.f;
  const float inv = ENERGY == CRL_ENERGY_COS ? a_stat[w] : 0.f;
  const float osc = g.pre ? 1.f : inv;                   // the final 1/|A_i| factor
  float pr = 0.f;
  for (int c = 0; c < D / 32; ++c) {
    const int k = lane + 32 * c;
    float v = 0.f;
    for (int s = 0; s < Sr; ++s) v += part[((size_t)s * Na + w) * D + k];
    if (ENERGY == CRL_ENERGY_L2) v += diag * (av[c] - bv[c]) - rs * av[c];
    if (ENERGY == CRL_ENERGY_DOT) v -= Cdiag * bv[c];
    if (ENERGY == CRL_ENERGY_COS) {
      v -= Cdiag * invb * (g.pre ? inv : 1.f) * bv[c];
      pr = fmaf(v, av[c] * inv, pr);
    }
    acc[c] = v;
  }
  if (ENERGY == CRL_ENERGY_COS) pr = warp_sum(pr);
  for (int c = 0; c < D / 32; ++c) {
    const int k = lane + 32 * c;
    float v = acc[c];
    if (ENERGY == CRL_ENERGY_COS) {
      const float u = av[c] * inv;
      v = inv < 1.f / kEpsCos ? (v - pr * u) * osc : v * osc;
    }
    out[(size_t)w * D + k] = v;
    outb[(size_t)w * D + k] = __float2bfloat16_rn(v);
  }
}

}  // namespace tc
}  // namespace crl
