// tc_merge.cuh — the per-row merge of split gradient partials (shared by the two-call logits
// kernels, tc_logits.cu, and the fused gradient pass, tc_gradf.cu).
//
// dA[i] = sum_s part[s][i]  (+ energy finalisation), fp32 and bf16 outputs.  One warp per row;
// D in {64, 128, 256} (every caller's representation size).
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
  const unsigned char* valid1 = nullptr;   // tc_grad2: per 128-row block, the extra slots holding data
  int prs_sub = 1;                         // row-sum sub-partials per slot (tc_grad2: 2 warpgroups)
};

// The loss reduced by the row-side merge (the D = 256 pair gradient path: one launch less):
// per row i the positive-pair logit l_ii from the same bf16 rows the logits used, and
// (LSE_i - l_ii, LSE'_i - l_ii, LSE_i^2); per-CTA partials, the last CTA (ticket) adds them in
// CTA order and finalises as the loss kernel does.  part == nullptr: off.
struct MergeLoss {
  const float* lr = nullptr;               // [Na] LSE_i of this rank's rows
  const float* lc = nullptr;               // [Na] LSE'_i of this rank's columns
  float* part = nullptr;                   // [CTAs][4]
  unsigned* ticket = nullptr;              // zero on entry, re-armed by the last CTA
  float* acc = nullptr;                    // [3] the sums (all-reduced by the caller at W > 1)
  float* out = nullptr;                    // [4] L_fwd, L_bwd, penalty, total (or null)
  int* skip = nullptr; int* adam_t = nullptr; int* status = nullptr;
  float invN = 0.f, c_f = 1.f, c_b = 1.f, beta = 0.f;
  int finalize = 1;                        // W = 1: finalise here; W > 1: the caller does
};



// V consecutive floats / bf16 of a row from lane-contiguous addresses (16 B vector accesses)
template <int V>
__device__ __forceinline__ void ld_f32v(const float* __restrict__ p, float (&v)[V]) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V / 4; ++i) {
      const float4 q = reinterpret_cast<const float4*>(p)[i];
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  } else {
    const float2 q = *reinterpret_cast<const float2*>(p);
    v[0] = q.x; v[1] = q.y;
  }
}
template <int V>
__device__ __forceinline__ void ld_bf16v(const __nv_bfloat16* __restrict__ p, float (&v)[V]) {
  uint32_t w[V / 2];
  if constexpr (V == 8) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
  } else if constexpr (V == 4) {
    const uint2 q = *reinterpret_cast<const uint2*>(p);
    w[0] = q.x; w[1] = q.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
#pragma unroll
  for (int i = 0; i < V / 2; ++i) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}

// One warp per row, lane l owns elements [V l, V l + V) (V = D / 32): every global access is a
// 16 B (8 B, 4 B) vector and all loads of the row are in flight before the first reduction.
template <int ENERGY, int V>
__device__ __forceinline__ void grad_merge_row_v(const GradMergeArgs& g, int w, int lane) {
  constexpr int D = 32 * V;
  const int row_offset = g.row_offset, Na = g.Na, S = g.S;
  if (w >= Na) return;
  const size_t ib = (size_t)(row_offset + w) * D + V * lane;
  // slots that hold data for this row (tc_grad2: the second slot only for cut row blocks)
  const int Sr = g.valid1 != nullptr ? min(S, 1 + (int)g.valid1[w >> 7]) : S;
  float av[V], bv[V], acc[V];
  ld_bf16v<V>(g.A + (size_t)w * D + V * lane, av);
  ld_bf16v<V>(g.Bg + ib, bv);
  ld_f32v<V>(g.part + (size_t)w * D + V * lane, acc);
  for (int s = 1; s < Sr; ++s) {
    float t[V];
    ld_f32v<V>(g.part + ((size_t)s * Na + w) * D + V * lane, t);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] += t[i];
  }
  constexpr bool DIFF = ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ;   // -(sum_j w_ij) A_i form
  float rs = 0.f;
  if (DIFF)
    for (int s = 0; s < Sr * g.prs_sub; ++s) rs += g.prs[(size_t)s * Na + w];
  const float Cdiag = g.Cdiag;
  float d2 = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const float d = av[i] - bv[i];
    d2 = fmaf(d, d, d2);
  }
  float diag = 0.f;                                      // energy-chain weight of the delta term
  if (ENERGY == CRL_ENERGY_L2) diag = Cdiag / sqrtf(warp_sum(d2) + kEpsL2);   // times (A_i - B_i)
  if (ENERGY == CRL_ENERGY_L2SQ) diag = 2.f * Cdiag;                            // L2^2: dl/dA = -2 (A - B)
  const float invb = ENERGY == CRL_ENERGY_COS ? g.b_stat[row_offset + w] : 0.f;
  const float inv = ENERGY == CRL_ENERGY_COS ? g.a_stat[w] : 0.f;
  const float osc = g.pre ? 1.f : inv;                   // the final 1/|A_i| factor
  float pr = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    float v = acc[i];
    if (DIFF) v += diag * (av[i] - bv[i]) - rs * av[i];
    if (ENERGY == CRL_ENERGY_DOT) v -= Cdiag * bv[i];
    if (ENERGY == CRL_ENERGY_COS) {
      v -= Cdiag * invb * (g.pre ? inv : 1.f) * bv[i];
      pr = fmaf(v, av[i] * inv, pr);
    }
    acc[i] = v;
  }
  if (ENERGY == CRL_ENERGY_COS) pr = warp_sum(pr);
  uint32_t hb[V / 2];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    float v = acc[i];
    if (ENERGY == CRL_ENERGY_COS) {
      const float u = av[i] * inv;
      v = inv < 1.f / kEpsCos ? (v - pr * u) * osc : v * osc;
    }
    acc[i] = v;
  }
#pragma unroll
  for (int i = 0; i < V / 2; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    hb[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  float* out = g.out + (size_t)w * D + V * lane;
  __nv_bfloat16* outb = g.outb + (size_t)w * D + V * lane;
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V / 4; ++i)
      reinterpret_cast<float4*>(out)[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
  } else {
    *reinterpret_cast<float2*>(out) = make_float2(acc[0], acc[1]);
  }
  if constexpr (V == 8) *reinterpret_cast<uint4*>(outb) = make_uint4(hb[0], hb[1], hb[2], hb[3]);
  else if constexpr (V == 4) *reinterpret_cast<uint2*>(outb) = make_uint2(hb[0], hb[1]);
  else *reinterpret_cast<uint32_t*>(outb) = hb[0];
}

template <int ENERGY>
__device__ __forceinline__ void grad_merge_row(const GradMergeArgs& g, int w, int lane) {
  if (g.D == 256) grad_merge_row_v<ENERGY, 8>(g, w, lane);
  else if (g.D == 128) grad_merge_row_v<ENERGY, 4>(g, w, lane);
  else grad_merge_row_v<ENERGY, 2>(g, w, lane);
}

// l_ii of row w (warp-uniform): the energy of (A_w, B_{row_offset + w}) on the bf16 rows
template <int ENERGY, int V>
__device__ __forceinline__ float merge_diag_logit(const GradMergeArgs& g, int w, int lane) {
  constexpr int D = 32 * V;
  float av[V], bv[V];
  ld_bf16v<V>(g.A + (size_t)w * D + V * lane, av);
  ld_bf16v<V>(g.Bg + (size_t)(g.row_offset + w) * D + V * lane, bv);
  float x = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) { const float d = av[i] - bv[i]; x = fmaf(d, d, x); }
    else x = fmaf(av[i], bv[i], x);
  }
  x = warp_sum(x);
  if (ENERGY == CRL_ENERGY_L2) return -sqrtf(x + kEpsL2);
  if (ENERGY == CRL_ENERGY_L2SQ) return -x;
  if (ENERGY == CRL_ENERGY_COS) return x * g.a_stat[w] * g.b_stat[g.row_offset + w];   // 1/|A_i|, 1/|B_i|
  return x;
}

}  // namespace tc
}  // namespace crl
