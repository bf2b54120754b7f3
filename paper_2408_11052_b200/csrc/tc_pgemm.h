// tc_pgemm.h — persistent CTA-pair GEMM (tc_pgemm.cu) for the wide encoder layers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace crl {
namespace tc {

enum PgemmEpi { PG_FWD_HIDDEN = 0, PG_FWD_OUT = 1, PG_DX = 2 };

// Tensor maps (bf16 unless stated, SWIZZLE_128B), built once at context creation:
//   a    : A operand {K, M}, box {64, 128}        (X for the forward, dZ for dX)
//   b    : forward: W {N = out, K = in}, box {64, 64};  dX: W {K = out, N = in}, box {64, 128}
//   out0 : hidden: Z {N, M}; output layer: Y fp32 {N, M} box {32, 32}; dX: dZ_prev {N, M}
//   out1 : hidden: act(Z) {N, M}; output layer: Y bf16 {N, M}                 (box {64, 32})
//   zin  : dX: Z_prev {N, M}, box {64, 32}
struct PgemmMaps {
  CUtensorMap a, b, out0, out1, zin;
};
struct PgemmArgs {
  int M, N, K;
  const float* bias;   // forward: [N]
  int act;             // crl_activation
  float* stat;         // output layer (N <= 256): row statistic of bf16(Y) (L2: |y|^2, cos: 1/|y|)
  int stat_energy;
  int dbg;             // measurement ablations (scratch/pgemm_test.cu); 0 in the library
  int lin;             // hidden: Z only (LayerNorm follows in its own kernel), no act(Z)
  long long* trace;    // development timestamps (scratch/pgemm_test.cu); nullptr in the library
};

// Up to two independent problems (the phi and psi encoders' same layer) in ONE persistent
// launch: the pairs walk problem 0's tiles, then problem 1's (one wave quantisation, not two)
struct PgemmJob {
  PgemmMaps maps[2];
  PgemmArgs args[2];
  int np, nt0, total;   // problems, tiles of problem 0, all tiles
};

bool tc_pgemm_supported(int M, int N, int K);
// both problems share the epilogue kind and activation
cudaError_t tc_pgemm2(int epi, const PgemmMaps& maps0, const PgemmArgs& p0, const PgemmMaps& maps1,
                      const PgemmArgs& p1, int num_sms, cudaStream_t st);
cudaError_t tc_pgemm(int epi, const PgemmMaps& maps, const PgemmArgs& p, int num_sms, cudaStream_t st);

}  // namespace tc
}  // namespace crl
