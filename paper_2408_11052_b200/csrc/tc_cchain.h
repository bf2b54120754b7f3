// tc_cchain.h — argument blocks of the cluster-split MLP chain kernels (tc_cchain.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace crl {
namespace tc {

constexpr int kCChainMaxL = 8;

struct CChainLayer {              // one GEMM step of the chain
  int K, N;                       // contraction / output widths
  const float* bias;              // FWD
  __nv_bfloat16* out_z;           // FWD hidden: Z_l [M][N]
  __nv_bfloat16* out_act;         // FWD output step: Y bf16 [M][N]
  float* out_f;                   // FWD output step: Y fp32 [M][N]
  const __nv_bfloat16* zprev;     // BWD: Z_{l-1} [M][N]
};
struct CChainEnc {
  int L;                          // GEMM steps (FWD: depth + 1, BWD: depth)
  float* out_stat;                // FWD: row statistic of bf16(Y)
  CChainLayer layer[kCChainMaxL];
};
struct CChainMaps {
  CUtensorMap a0;                 // FWD: X0 {K0, M} box {64,128}; BWD: dY {D, M} box {64,128}
  CUtensorMap w[kCChainMaxL];     // W_l {out, in}, box {64, 64}
  CUtensorMap st[kCChainMaxL];    // TMA-store targets {N, M} box {64, 128}: FWD X_{l+1}, BWD dZ_{l-1}
};
struct CChainParams {
  int M, act, energy;
  int store_ok;                   // 1 (measurement knob: 0 skips the HBM stores)
  int trace;                      // measurement: globaltimer trace of cluster 0 (CRL_CCHAIN_TRACE)
  CChainEnc enc[2];
};

size_t tc_cchain_smem();
bool tc_cchain_supported(int in0, int width, int D, int depth);
cudaError_t tc_cchain_forward(const CChainMaps& m0, const CChainMaps& m1, const CChainParams& p, cudaStream_t st);
cudaError_t tc_cchain_backward(const CChainMaps& m0, const CChainMaps& m1, const CChainParams& p, cudaStream_t st);

}  // namespace tc
}  // namespace crl
