// tc_grad2.h — both-sides logits gradient pass at D = 256 (tc_grad2.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace crl {
namespace tc {

struct Grad2Side {
  const float* a_stat;          // [Na] row statistic of A (L2: |a|^2, cos: 1/|a|, bf16-rounded rows)
  const float* b_stat;          // [Nb + pad] column statistic of B
  const float* lr;              // [Na] LSE of this side's rows (natural log)
  const float* lc;              // [Nb + pad] LSE of the columns
  const float* lcf;             // [Nb + pad] column factor 2^(-lc log2 e)(invN c_c + 2 invN beta_c lc)
  float c_r, c_c, beta_r, beta_c;
  float* part_da;               // [2][Na][256] dA partial slots (slot 1: second piece of a cut row block)
  float* part_rs;               // [2 slots][2 warpgroups][Na] row sums of w (L2)
  const __nv_bfloat16* A;       // [Na][256] bf16 rows (held in TMEM per row block)
};
struct Grad2Args {
  int Na, Nb;                   // rows per side (local batch), columns (global batch)
  int RB, TPB;                  // filled by tc_grad2: row blocks, 64-column tiles per row block
  float invN;
  const int* fac_ok;            // 1: every row / column factor of the step is a normal float
  Grad2Side side[2];            // 0: rows Phi, columns Psi (dPhi); 1: rows Psi, columns Phi (dPsi)
  int dbg;                      // measurement ablations (scratch/g2_bench.cu); 0 in the library
  int nsides;                   // tc_grad2p: 1 = side 0 only (W stored, side 1 by a GEMM); 0 / 2 = both
  int w_store;                  // tc_grad2p, nsides = 1: store W (bf16 [Na][Nb]) through the mW map
  unsigned long long* trace;    // measurement: CTA 0 event clocks [1024][8]; null in the library
};

int tc_grad2_grid(int Na, int num_sms);
void tc_grad2_split_flags(int Na, int Nb, int grid, unsigned char* flags);
cudaError_t tc_grad2(int energy, const CUtensorMap& mB0, const CUtensorMap& mB1, const Grad2Args& p, int grid,
                     cudaStream_t st);
// CTA-pair variant: D maps box {64, 128} (dA parts), S maps box {64, 64} (S parts); grid = 2 x pairs
int tc_grad2p_grid(int Na, int num_sms);
int tc_grad2p_warpgroups();                // epilogue warpgroups = L2 row-sum sub-slots per partial slot
// per 128-row block: the number of extra partial slots its pieces use (merge: 1 + flag slots);
// returns the most slots any row block uses
int tc_grad2p_split_flags(int Na, int Nb, int grid, unsigned char* flags, int nsides = 2);
// mA0 / mA1: the LOCAL rows of each side (Phi, Psi bf16 [Na][256]), box {64, 128}.
// mW (p.w_store = 1, p.nsides = 1): W = dL/dS (the bf16 weights of the side-0 dA MMA) as bf16
// [Na][Nb], box {64, 128}, SW128; the symmetric energies (L2, L2^2, dot) give side 1's weights as
// W^T, so dPsi = W^T Phi (+ the L2 column sums of W) is a plain GEMM (tc_pdw.h pdw_add_gemm).
cudaError_t tc_grad2p(int energy, const CUtensorMap& mD0, const CUtensorMap& mD1, const CUtensorMap& mS0,
                      const CUtensorMap& mS1, const CUtensorMap& mA0, const CUtensorMap& mA1, const Grad2Args& p,
                      int grid, cudaStream_t st, const CUtensorMap* mW = nullptr);

}  // namespace tc
}  // namespace crl
