// tc_chain.h — argument blocks of the fused MLP chain kernels (tc_chain.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

namespace crl {
namespace tc {

constexpr int kChainMaxL = 8;

struct ChainLayer {
  int K, N;                       // contraction / output widths of this GEMM step
  const float* bias;              // FWD
  __nv_bfloat16* out_act;         // FWD hidden: X_{l+1}; FWD last: Y bf16; BWD: dZ_{l-1}   ([M][N])
  __nv_bfloat16* out_z;           // FWD hidden: Z_l
  const __nv_bfloat16* zprev;     // BWD: Z_{l-1}
  float* out_f;                   // FWD last: Y fp32
};
struct ChainEnc {
  int L;
  float* out_stat;                // FWD: row statistic of Y (bf16-rounded)
  ChainLayer layer[kChainMaxL];
};
struct ChainMaps {
  CUtensorMap a0;                 // FWD: X0 {K0, M} box {64,128};  BWD: dY {D, M} box {64,128}
  CUtensorMap w[kChainMaxL];      // FWD: W_l MN-major {out, in} box {64,64}; BWD: K-major {out, in} box {64, in}
  CUtensorMap st_out[kChainMaxL]; // TMA-store targets, box {64,128}: FWD X_{l+1} / Y bf16, BWD dZ_{l-1}
  CUtensorMap st_z[kChainMaxL];   // FWD hidden: Z_l, box {64,128}
};
struct ChainParams {
  int M, act, energy;
  int* fac_ok;                    // FWD: re-armed to fac_init by block (0,0) (see tc_logits.cu)
  int fac_init;
  int dbg;                        // measurement knob (CRL_CHAIN_DBG): 1 = no global stores, 2 = no epilogue math
  ChainEnc enc[2];
};

size_t tc_chain_smem();
bool tc_chain_supported(int in0, int width, int D, int depth);
cudaError_t tc_chain_forward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st);
cudaError_t tc_chain_backward(const ChainMaps& m0, const ChainMaps& m1, const ChainParams& p, cudaStream_t st);

}  // namespace tc
}  // namespace crl
