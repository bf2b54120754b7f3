// tc_pdw.h — weight / bias gradients of the wide encoders on CTA pairs (tc_pdw.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace crl {
namespace tc {

constexpr int kPdwMaxProblems = 16;

struct alignas(64) PdwProblem {
  CUtensorMap a;           // X_l  [K][ldx] bf16, box {64, 64}: the MN-major A operand (M = in)
  CUtensorMap b;           // dZ_l [K][N]   bf16, box {64, 64}: the MN-major B operand
  CUtensorMap out;         // dW_l partial slices fp32 [S][M][N], box {32, 32, 1} (TMA stores)
  float* db;               // db_l slice 0 ([N]; slice s at + s * db_stride), or null
  long long db_stride;     // floats between the db slices (the parameter count for dW / db)
  int out_t;               // 1: out is stored transposed, [S][N][M] (pdw_add_gemm_t)
  int M, N;                // dW_l is [M = in][N = out]
  int tiles_n, tiles;      // 256 x 256 nh tiles per slice along N; work items = tiles_m * tiles_n * S
};

struct PdwParams {
  PdwProblem prob[kPdwMaxProblems];
  int n, total;            // problems, work items
  int K, splits, kb_per_split;
  long long split_stride;  // floats between partial slices (the parameter count)
  int dbg;                 // measurement ablations (env CRL_PDW_DBG): 1 no bias reads, 2 no MMA, 4 no TMA
  int nh;                  // 256-column halves per item: 2 (256 x 512 tiles, default) or 1 (CRL_PDW_NH=1)
};

void pdw_init(PdwParams& P, int K, int splits, size_t split_stride);
// X: [K][ldx] bf16 (ldx >= M), dZ: [K][N] bf16, dW / db: slice-0 destinations in the gradient
// buffer.  Returns false when a tensor map cannot be encoded or the table is full.
bool pdw_add_problem(PdwParams& P, const __nv_bfloat16* X, int ldx, const __nv_bfloat16* dZ, int M, int N,
                     float* dW, float* db);
// The same engine as a general GEMM with a TRANSPOSED result: out_t[N][M] (fp32 slices
// [S][N][M], out_stride floats apart) = (sum_K A[K][M] B[K][N])^T, and colsum_b[N] (slices
// colsum_stride apart, or null) = sum_K B[K][N].  A: [K][lda] bf16, B: [K][ldb] bf16 (M, N
// contiguous).  Used for dPsi = W^T Phi (A = Phi, B = the stored W: out_t = dPsi partials
// [N][256], row-major like every other partial).
bool pdw_add_gemm_t(PdwParams& P, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, int ldb, int M, int N,
                    float* out_t, long long out_stride, float* colsum_b, long long colsum_stride);
void pdw_set_nh(PdwParams& P, int nh);
bool pdw_supported(int K, int splits);
cudaError_t tc_pdw_launch(const PdwParams& P, int num_sms, cudaStream_t st);

}  // namespace tc
}  // namespace crl
