// logits_simt.cu — fp32 SIMT energy logits + online logsumexp (A3) and the in-pass
// dlogits -> representation gradients (A4).  The N x N logits are never stored.
//
// Paper: energies App. A.2 P:607-617 (L2 with the minus sign of P:614, reading A-01; dot
// P:610; cos P:608), InfoNCE fwd/bwd/sym P:619-630, logsumexp penalty P:361 / Alg. 1 P:1052.
// Readings A-02..A-06.
//
// Both kernels are "row-owner" kernels over an orientation (A rows, B columns):
//   l_ij = f(A_i, B_j)  (f is symmetric in its two arguments for L2 / dot / cos)
// * lse kernel : LSE_i = log sum_j exp(l_ij), online over column tiles.  Called with
//   (A,B) = (Phi, Psi) for the row LSE and with (Psi, Phi) for the column LSE'.
// * grad kernel: dA_i = sum_j g_ij df(A_i,B_j)/dA_i with the closed-form dlogits
//     g_ij = invN [c_r (e^{l-lr_i} - d_ij) + c_c (e^{l-lc_j} - d_ij)]
//            + 2 invN (beta_r lr_i e^{l-lr_i} + beta_c lc_j e^{l-lc_j})
//   formed in registers and consumed in the same pass (never written to HBM).  With
//   (A,B) = (Phi,Psi): lr = LSE, lc = LSE', (c_r,c_c) = (c_f,c_b), beta_r = beta.
//   With (A,B) = (Psi,Phi): lr = LSE', lc = LSE, (c_r,c_c) = (c_b,c_f), beta_c = beta.
//   Energy chain: dot w = g;  L2 w = g / r (r = -l) and dA_i = sum_j w_ij B_j - (sum_j w_ij) A_i;
//   cos w = g / |B_j|, du_i = sum_j w_ij B_j, dA_i = (du_i - (du_i.u_i) u_i) / |A_i|;
//   L2sq (F3) w = 2 g with the L2 form; L1 (F3) dA_ik = sum_j g_ij sign(B_jk - A_ik) (no
//   contraction form: an ALU pass over the same W tile, reading A-33 for ties).
// L2 uses the difference form sum_k (a_k - b_k)^2 (no cancellation) on this fp32 path.
//
// Tiling: TR (16/32/64) A-rows per CTA, 64 B-rows per column tile; A and the column tiles
// are held TRANSPOSED in shared memory ([k][row], odd pitch) so every read in both the
// logits and the dA contraction is conflict-free; column tiles are double-buffered with
// 4-byte cp.async.  Thread (tx,ty) owns rows ty+16i and columns tx+16j.
#include "common.cuh"
#include <math_constants.h>

namespace crl {

struct LogitsArgs {
  const float* A; int Na; int row_offset;   // global index of A row 0 (delta_ij)
  const float* B; int Nb;                   // B rows are global column indices 0..Nb-1
  const float* lr;                          // grad: row statistic [Na]
  const float* lc;                          // grad: column statistic [Nb]
  float c_r, c_c, beta_r, beta_c, invN;
  float* out;                               // lse: [Na]; grad: dA [Na][D]; pair stats: R [Na]
  // pairwise / FB losses (F3): per-PHI-index statistics (rows for orient 0, columns for 1)
  const float* pd = nullptr;                // diagonal l_kk
  const float* pR = nullptr;                // sum_{j != k} h(l_kj, d_k)      (DPO, IPO)
  const float* plse = nullptr;              // row logsumexp (penalty term)
  int orient = 0, loss = 0, Ntot = 0;
  float inv_nm1 = 0.f;                      // 1 / (N - 1)
  float* out2 = nullptr;                    // pair stats: per-row loss sums [Na]
};

// pairwise / FB losses (oracle/losses.py pairwise_grad): off-diagonal g = h / N, diagonal D / N
__device__ __forceinline__ float pair_h(int loss, float l, float d, float inv_nm1) {
  switch (loss) {
    case CRL_LOSS_FB: return __expf(2.f * l) * inv_nm1;
    case CRL_LOSS_DPO: return 1.f / (1.f + __expf(d - l));
    case CRL_LOSS_IPO: return 2.f * (l - d + 1.f);
    default: return 2.f * (l + 1.f);                              // SPPO
  }
}
__device__ __forceinline__ float pair_diag(int loss, float d, float R, int N) {
  switch (loss) {
    case CRL_LOSS_FB: return -__expf(d);
    case CRL_LOSS_DPO:
    case CRL_LOSS_IPO: return -R;
    default: return 2.f * (d + 1.f) + 2.f * (float)N * (d - 1.f);  // SPPO
  }
}
// the loss contribution of pair (i, j) (per-row extras -e^{d_i} (FB), N (d_i - 1)^2 (SPPO) are
// added by the loss kernel)
__device__ __forceinline__ float pair_term(int loss, float l, float d, bool diag, float inv_nm1) {
  switch (loss) {
    case CRL_LOSS_FB: return diag ? 0.f : 0.5f * inv_nm1 * __expf(2.f * l);
    case CRL_LOSS_DPO: { const float x = l - d; return fmaxf(x, 0.f) + log1pf(__expf(-fabsf(x))); }
    case CRL_LOSS_IPO: { const float x = d - l - 1.f; return x * x; }
    default: { const float x = l + 1.f; return x * x; }            // SPPO
  }
}

constexpr int TC = 64;                      // columns per tile
constexpr int BPITCH = TC + 1;

__device__ __forceinline__ void cpa4(float* smem, const float* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int D, int TR>
struct LSmem {
  static constexpr int AP = TR + 1;
  static constexpr size_t floats(bool grad) {
    return (size_t)D * AP + 2 * (size_t)D * BPITCH + TR + 2 * TC + (grad ? (size_t)TR * BPITCH : 0);
  }
};

template <int D, int TR, int ENERGY, bool GRAD, bool PAIR>
__global__ void __launch_bounds__(256) logits_rows_kernel(LogitsArgs p) {
  constexpr int AP = TR + 1;
  constexpr int RI = TR / 16;              // rows per thread
  constexpr int DC = D / 16;               // d-columns per thread in the dA accumulation
  extern __shared__ float sm[];
  float* At = sm;                          // [D][AP]      A^T
  float* Bt = At + D * AP;                 // [2][D][BPITCH]  B^T column tiles
  float* nA = Bt + 2 * D * BPITCH;         // [TR]  inverse clamped norms (cos)
  float* nB = nA + TR;                     // [2][TC]
  float* Ws = nB + 2 * TC;                 // [TR][BPITCH] (grad only)

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int a0 = blockIdx.x * TR;
  const int ntiles = (p.Nb + TC - 1) / TC;
  pdl_wait();
  pdl_launch();

  auto issue_b = [&](int buf, int b0) {
    float* dst = Bt + buf * D * BPITCH;
    for (int e = tid; e < TC * D; e += 256) {
      const int r = e / D, c = e - r * D;
      const bool ok = b0 + r < p.Nb;
      cpa4(dst + c * BPITCH + r, ok ? p.B + (size_t)(b0 + r) * D + c : p.B, ok);
    }
  };
  // A tile (transposed) + first column tile
  for (int e = tid; e < TR * D; e += 256) {
    const int r = e / D, c = e - r * D;
    const bool ok = a0 + r < p.Na;
    cpa4(At + c * AP + r, ok ? p.A + (size_t)(a0 + r) * D + c : p.A, ok);
  }
  issue_b(0, 0);
  cpa_commit();

  float lr_i[RI];
  float pd_i[RI], pl_i[RI], pR_i[RI];                     // PAIR: this row's phi-index stats (orient 0)
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int r = a0 + ty + 16 * i;
    lr_i[i] = (GRAD && !PAIR && r < p.Na) ? p.lr[r] : 0.0f;
    const bool own = PAIR && r < p.Na && p.orient == 0;
    pd_i[i] = own ? p.pd[p.row_offset + r] : 0.f;
    pl_i[i] = (own && GRAD) ? p.plse[p.row_offset + r] : 0.f;
    pR_i[i] = (own && GRAD && p.pR) ? p.pR[p.row_offset + r] : 0.f;
  }
  float m_run[RI], s_run[RI], wsum[RI];
  float acc2[RI][GRAD ? DC : 1];
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    m_run[i] = PAIR ? 0.f : -CUDART_INF_F; s_run[i] = 0.f; wsum[i] = 0.f;
#pragma unroll
    for (int c = 0; c < (GRAD ? DC : 1); ++c) acc2[i][c] = 0.f;
  }

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1, b0 = t * TC;
    if (t + 1 < ntiles) {
      issue_b(buf ^ 1, b0 + TC);
      cpa_commit();
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const float* B_ = Bt + buf * D * BPITCH;
    if (ENERGY == CRL_ENERGY_COS) {
      if (t == 0 && tid < TR) {
        float s = 0.f;
        for (int c = 0; c < D; ++c) s = fmaf(At[c * AP + tid], At[c * AP + tid], s);
        nA[tid] = 1.0f / fmaxf(sqrtf(s), kEpsCos);
      }
      if (tid >= 128 && tid < 128 + TC) {
        const int r = tid - 128;
        float s = 0.f;
        for (int c = 0; c < D; ++c) s = fmaf(B_[c * BPITCH + r], B_[c * BPITCH + r], s);
        nB[buf * TC + r] = 1.0f / fmaxf(sqrtf(s), kEpsCos);
      }
      __syncthreads();
    }

    // ---- RI x 4 logits per thread
    float acc[RI][4];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
    for (int k = 0; k < D; ++k) {
      float a[RI], b[4];
#pragma unroll
      for (int i = 0; i < RI; ++i) a[i] = At[k * AP + ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = B_[k * BPITCH + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) {
            const float d = a[i] - b[j];
            acc[i][j] = fmaf(d, d, acc[i][j]);
          } else if (ENERGY == CRL_ENERGY_L1) {
            acc[i][j] += fabsf(a[i] - b[j]);
          } else {
            acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          }
        }
    }
    bool valid[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) valid[j] = (b0 + tx + 16 * j) < p.Nb;
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v = acc[i][j];
        if (ENERGY == CRL_ENERGY_L2) v = -sqrtf(v + kEpsL2);
        if (ENERGY == CRL_ENERGY_L2SQ || ENERGY == CRL_ENERGY_L1) v = -v;
        if (ENERGY == CRL_ENERGY_COS) v = v * nA[ty + 16 * i] * nB[buf * TC + tx + 16 * j];
        acc[i][j] = v;                    // acc now holds l_ij
      }

    if (PAIR && !GRAD) {
      // pair statistics of this row: m_run <- sum_{j != i} h, s_run <- sum_j loss term
#pragma unroll
      for (int i = 0; i < RI; ++i) {
        const int ig = p.row_offset + a0 + ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!valid[j]) continue;
          const int jg = b0 + tx + 16 * j;
          const bool dg = ig == jg;
          if (!dg) m_run[i] += pair_h(p.loss, acc[i][j], pd_i[i], p.inv_nm1);
          s_run[i] += pair_term(p.loss, acc[i][j], pd_i[i], dg, p.inv_nm1);
        }
      }
    } else if (!GRAD) {
#pragma unroll
      for (int i = 0; i < RI; ++i) {
        float mx = m_run[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) if (valid[j]) mx = fmaxf(mx, acc[i][j]);
        if (mx == -CUDART_INF_F) continue;
        float s = s_run[i] * expf(m_run[i] - mx);     // m_run = -inf -> 0
#pragma unroll
        for (int j = 0; j < 4; ++j) if (valid[j]) s += expf(acc[i][j] - mx);
        s_run[i] = s; m_run[i] = mx;
      }
    } else {
      // ---- dlogits in registers -> energy chain -> W tile in shared memory
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int jg = b0 + tx + 16 * j;
        const float lcj = valid[j] ? p.lc[jg] : 0.f;
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          const int ig = p.row_offset + a0 + ty + 16 * i;
          float w = 0.f;
          if (valid[j]) {
            const float lv = acc[i][j];
            float g;
            if (PAIR) {
              // phi index of the pair: the row (orient 0) or the column (orient 1)
              const bool o1 = p.orient != 0;
              const float d = o1 ? p.pd[jg] : pd_i[i];
              const float ls = o1 ? p.plse[jg] : pl_i[i];
              const float gp = (ig != jg) ? pair_h(p.loss, lv, d, p.inv_nm1)
                                          : pair_diag(p.loss, d, o1 ? (p.pR ? p.pR[jg] : 0.f) : pR_i[i], p.Ntot);
              g = p.invN * gp + 2.f * p.invN * p.beta_r * ls * expf(lv - ls);
            } else {
              const float pe = expf(lv - lr_i[i]);
              const float qe = expf(lv - lcj);
              const float dlt = (ig == jg) ? 1.f : 0.f;
              g = p.invN * (p.c_r * (pe - dlt) + p.c_c * (qe - dlt)) +
                  2.f * p.invN * (p.beta_r * lr_i[i] * pe + p.beta_c * lcj * qe);
            }
            if (ENERGY == CRL_ENERGY_L2) w = g / (-lv);
            else if (ENERGY == CRL_ENERGY_L2SQ) w = 2.f * g;
            else if (ENERGY == CRL_ENERGY_COS) w = g * nB[buf * TC + tx + 16 * j];
            else w = g;
          }
          Ws[(ty + 16 * i) * BPITCH + tx + 16 * j] = w;
          if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) wsum[i] += w;
        }
      }
      __syncthreads();
      // dA[rows][d] += W[rows][64] . B[64][d]
#pragma unroll 4
      for (int jj = 0; jj < TC; ++jj) {
        float w[RI];
#pragma unroll
        for (int i = 0; i < RI; ++i) w[i] = Ws[(ty + 16 * i) * BPITCH + jj];
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          const float bv = B_[(tx + 16 * c) * BPITCH + jj];
#pragma unroll
          for (int i = 0; i < RI; ++i) {
            if (ENERGY == CRL_ENERGY_L1) {
              const float d = bv - At[(tx + 16 * c) * AP + ty + 16 * i];
              const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
              acc2[i][c % (GRAD ? DC : 1)] = fmaf(w[i], sg, acc2[i][c % (GRAD ? DC : 1)]);
            } else {
              acc2[i][c % (GRAD ? DC : 1)] = fmaf(w[i], bv, acc2[i][c % (GRAD ? DC : 1)]);
            }
          }
        }
      }
    }
    __syncthreads();                       // buffer `buf` is refilled two tiles later
  }

  if (PAIR && !GRAD) {
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      float R = m_run[i], Lr = s_run[i];
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        R += __shfl_xor_sync(0xffffffffu, R, o);
        Lr += __shfl_xor_sync(0xffffffffu, Lr, o);
      }
      const int r = a0 + ty + 16 * i;
      if (tx == 0 && r < p.Na) { p.out[r] = R; p.out2[r] = Lr; }
    }
  } else if (!GRAD) {
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      float m = m_run[i], s = s_run[i];
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mx = fmaxf(m, m2);
        const float t = (m == -CUDART_INF_F ? 0.f : s * expf(m - mx)) +
                        (m2 == -CUDART_INF_F ? 0.f : s2 * expf(m2 - mx));
        m = mx; s = t;
      }
      const int r = a0 + ty + 16 * i;
      if (tx == 0 && r < p.Na) p.out[r] = m + logf(s);
    }
  } else {
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      const int rl = ty + 16 * i;
      const int r = a0 + rl;
      float* acc_i = acc2[i];
      if (ENERGY == CRL_ENERGY_L2 || ENERGY == CRL_ENERGY_L2SQ) {
        float ws = wsum[i];
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
#pragma unroll
        for (int c = 0; c < DC; ++c) acc_i[c % (GRAD ? DC : 1)] -= ws * At[(tx + 16 * c) * AP + rl];
      } else if (ENERGY == CRL_ENERGY_COS) {
        const float inv = nA[rl];
        float pr = 0.f;
#pragma unroll
        for (int c = 0; c < DC; ++c) pr = fmaf(acc_i[c % (GRAD ? DC : 1)], At[(tx + 16 * c) * AP + rl], pr);
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
        pr *= inv;                                        // du . u
        const bool big = inv < 1.0f / kEpsCos;           // ||A_i|| > eps
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          const float u = At[(tx + 16 * c) * AP + rl] * inv;
          float& v = acc_i[c % (GRAD ? DC : 1)];
          v = big ? (v - pr * u) * inv : v * inv;
        }
      }
      if (r < p.Na) {
#pragma unroll
        for (int c = 0; c < DC; ++c) p.out[(size_t)r * D + tx + 16 * c] = acc_i[c % (GRAD ? DC : 1)];
      }
    }
  }
}

static int g_sms_logits = 148;
void logits_set_num_sms(int n) { g_sms_logits = n > 0 ? n : 148; }

template <int D, int TR, int ENERGY, bool GRAD, bool PAIR = false>
static cudaError_t launch_logits_t(const LogitsArgs& p, cudaStream_t st) {
  const size_t smem = sizeof(float) * LSmem<D, TR>::floats(GRAD);
  static bool attr_set = false;   // per template instance
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(logits_rows_kernel<D, TR, ENERGY, GRAD, PAIR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((p.Na + TR - 1) / TR);
  return launch_pdl(logits_rows_kernel<D, TR, ENERGY, GRAD, PAIR>, grid, dim3(256), smem, st, p);
}

template <int D, int ENERGY, bool GRAD>
static cudaError_t launch_logits_tr(const LogitsArgs& p, cudaStream_t st) {
  if (p.loss >= CRL_LOSS_FB) return launch_logits_t<D, 16, ENERGY, GRAD, true>(p, st);   // F3 pair losses
  if (p.Na >= 64 * g_sms_logits) return launch_logits_t<D, 64, ENERGY, GRAD>(p, st);
  if (p.Na >= 16 * g_sms_logits) return launch_logits_t<D, 32, ENERGY, GRAD>(p, st);
  return launch_logits_t<D, 16, ENERGY, GRAD>(p, st);
}

template <int D, bool GRAD>
static cudaError_t launch_logits_e(int energy, const LogitsArgs& p, cudaStream_t st) {
  switch (energy) {
    case CRL_ENERGY_L2: return launch_logits_tr<D, CRL_ENERGY_L2, GRAD>(p, st);
    case CRL_ENERGY_DOT: return launch_logits_tr<D, CRL_ENERGY_DOT, GRAD>(p, st);
    case CRL_ENERGY_COS: return launch_logits_tr<D, CRL_ENERGY_COS, GRAD>(p, st);
    case CRL_ENERGY_L1: return launch_logits_tr<D, CRL_ENERGY_L1, GRAD>(p, st);
    case CRL_ENERGY_L2SQ: return launch_logits_tr<D, CRL_ENERGY_L2SQ, GRAD>(p, st);
  }
  return cudaErrorInvalidValue;
}

template <bool GRAD>
static cudaError_t launch_logits_d(int D, int energy, const LogitsArgs& p, cudaStream_t st) {
  switch (D) {
    case 16: return launch_logits_e<16, GRAD>(energy, p, st);
    case 32: return launch_logits_e<32, GRAD>(energy, p, st);
    case 64: return launch_logits_e<64, GRAD>(energy, p, st);
    case 128: return launch_logits_e<128, GRAD>(energy, p, st);
    case 256: return launch_logits_e<256, GRAD>(energy, p, st);
  }
  return cudaErrorInvalidValue;
}

bool logits_simt_supports(int D) { return D == 16 || D == 32 || D == 64 || D == 128 || D == 256; }

cudaError_t logits_lse_f32(int D, int energy, const float* A, int Na, const float* B, int Nb,
                           float* lse_out, cudaStream_t st) {
  LogitsArgs p{};
  p.A = A; p.Na = Na; p.B = B; p.Nb = Nb; p.out = lse_out;
  return launch_logits_d<false>(D, energy, p, st);
}

cudaError_t logits_grad_f32(int D, int energy, const float* A, int Na, int row_offset,
                            const float* B, int Nb, const float* lr, const float* lc, float c_r,
                            float c_c, float beta_r, float beta_c, float invN, float* dA,
                            cudaStream_t st) {
  LogitsArgs p{};
  p.A = A; p.Na = Na; p.row_offset = row_offset; p.B = B; p.Nb = Nb;
  p.lr = lr; p.lc = lc; p.c_r = c_r; p.c_c = c_c; p.beta_r = beta_r; p.beta_c = beta_c;
  p.invN = invN; p.out = dA;
  return launch_logits_d<true>(D, energy, p, st);
}



// F3 pair / FB losses.  Row statistics (orient 0, A = Phi rows, B = Psi): R_i = sum_{j != i}
// h(l_ij, d_i), Lrow_i = sum_j (loss term); d = the diagonal l_kk (global, [N]).
cudaError_t logits_pair_stats_f32(int D, int energy, int loss, const float* A, int Na, int row_offset,
                                  const float* B, int Nb, const float* diag, float* R_out, float* L_out,
                                  cudaStream_t st) {
  LogitsArgs p{};
  p.A = A; p.Na = Na; p.row_offset = row_offset; p.B = B; p.Nb = Nb; p.out = R_out; p.out2 = L_out;
  p.pd = diag; p.loss = loss; p.Ntot = Nb; p.inv_nm1 = Nb > 1 ? 1.f / (float)(Nb - 1) : 1.f;
  return launch_logits_d<false>(D, energy, p, st);
}
// dA for a pair / FB loss: orient 0: (A, B) = (Phi, Psi); orient 1: (A, B) = (Psi, Phi).
// diag / R / lse are indexed by the Phi index (global, [N]); beta = the row-LSE penalty weight.
cudaError_t logits_pair_grad_f32(int D, int energy, int loss, int orient, const float* A, int Na, int row_offset,
                                 const float* B, int Nb, const float* diag, const float* R, const float* lse,
                                 float beta, float invN, float* dA, cudaStream_t st) {
  LogitsArgs p{};
  p.A = A; p.Na = Na; p.row_offset = row_offset; p.B = B; p.Nb = Nb; p.out = dA;
  p.pd = diag; p.pR = R; p.plse = lse; p.orient = orient; p.loss = loss; p.Ntot = Nb;
  p.inv_nm1 = Nb > 1 ? 1.f / (float)(Nb - 1) : 1.f;
  p.beta_r = beta; p.invN = invN;
  return launch_logits_d<true>(D, energy, p, st);
}

}  // namespace crl
