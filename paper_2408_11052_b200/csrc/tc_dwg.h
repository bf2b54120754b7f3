// tc_dwg.h — argument block of the grouped weight/bias-gradient kernel (tc_dwg.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace crl {
namespace tc {

constexpr int kDwgMaxProblems = 16;

struct DwgProblem {
  CUtensorMap mapX;        // X_l  [K][ldx] bf16, box {64, 64}
  CUtensorMap mapDZ;       // dZ_l [K][N]   bf16, box {64, 64}
  CUtensorMap mapW;        // dW_l partials [splits][M][N] fp32, box {32, 128, 1} (TMA-store epilogue)
  int M, N;                // dW_l is [M = in][N = out]
  int bn;                  // columns per tile (multiple of 64, <= 256)
  int mblk, nblk, tiles;   // tiles = mblk * nblk * splits
  int tma_w;               // dW tile leaves through SMEM staging + TMA stores (16 B aligned rows)
  float* dW;               // slice 0 of the split-K partials (slice s at + s * split_stride)
  float* db;               // same, [N]
};

struct DwgParams {
  DwgProblem prob[kDwgMaxProblems];
  int n, total_tiles;
  int K, splits, k_per_split;
  size_t split_stride;
};

void dwg_init(DwgParams& P, int K, int splits, size_t split_stride);
bool dwg_add_problem(DwgParams& P, const __nv_bfloat16* X, int ldx, const __nv_bfloat16* dZ, int M, int N,
                     float* dW, float* db);
cudaError_t tc_dwg_launch(const DwgParams& P, cudaStream_t st);

}  // namespace tc
}  // namespace crl
