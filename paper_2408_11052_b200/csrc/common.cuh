// common.cuh — shared device/host helpers for the CRL hot path (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstddef>

#include "crl.h"

#define CRL_MAX_LAYERS 8

namespace crl {

// ---------------------------------------------------------------------------------------
// Host-side plan of one encoder: layer l has W[in][out] at w_off and b[out] at b_off in the
// flat parameter buffer (include/crl.h layout).
// ---------------------------------------------------------------------------------------
struct LayerPlan { int in, out; size_t w_off, b_off, g_off, be_off; };   // g/be: LayerNorm (F2)
struct EncoderPlan {
  int n_layers;          // depth hidden + 1 output
  int in_dim;
  size_t param_off, n_params;
  LayerPlan layer[CRL_MAX_LAYERS];
};

// hidden layers: W, b (+ LayerNorm gamma, beta when `ln`); output layer: W, b
inline EncoderPlan make_encoder_plan(int in_dim, int depth, int width, int out_dim, size_t off, bool ln = false) {
  EncoderPlan p{};
  p.n_layers = depth + 1;
  p.in_dim = in_dim;
  p.param_off = off;
  int prev = in_dim;
  for (int l = 0; l <= depth; ++l) {
    int o = (l < depth) ? width : out_dim;
    p.layer[l].in = prev;
    p.layer[l].out = o;
    p.layer[l].w_off = off;
    off += (size_t)prev * o;
    p.layer[l].b_off = off;
    off += o;
    if (ln && l < depth) {
      p.layer[l].g_off = off;
      off += o;
      p.layer[l].be_off = off;
      off += o;
    }
    prev = o;
  }
  p.n_params = off - p.param_off;
  return p;
}

// ---------------------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }
__device__ __forceinline__ float silu_grad_f(float z) {
  float s = 1.0f / (1.0f + __expf(-z));
  return s * (1.0f + z * (1.0f - s));
}
__device__ __forceinline__ float act_f(float z, int act) {
  return act == CRL_ACT_SILU ? silu_f(z) : fmaxf(z, 0.0f);
}
__device__ __forceinline__ float act_grad_f(float z, int act) {
  return act == CRL_ACT_SILU ? silu_grad_f(z) : (z > 0.0f ? 1.0f : 0.0f);
}

// Status word handling: first fault wins.
__device__ __forceinline__ void set_status(int* status, int code) {
  atomicCAS(status, 0, code);
}

constexpr float kEpsL2 = 1e-12f;   // reading A-06
constexpr float kEpsCos = 1e-8f;

// ---------------------------------------------------------------------------------------
// Programmatic dependent launch: every kernel of the step is launched with
// programmaticStreamSerialization, waits for its predecessor's memory with
// griddepcontrol.wait before touching predecessor-produced data, and lets its own
// dependents start their prologue early (griddepcontrol.launch_dependents).  Without the
// launch attribute both instructions are no-ops.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace crl
