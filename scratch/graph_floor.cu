// Calibration: per-kernel latency of a chain of dependent tiny kernels in a CUDA graph,
// with and without programmatic dependent launch (measurement only, not part of the build).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(float* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) x[blockIdx.x] += 1.f;
}
int main() {
  float* x; cudaMalloc(&x, 4096 * 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int blocks : {1, 8, 148}) {
      const int K = 32;
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < K; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(128); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, tiny, x, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a, s);
      const int R = 200;
      for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("pdl=%d blocks=%d: %.2f us per graph of %d kernels = %.2f us/kernel\n", pdl, blocks, ms * 1e3 / R, K,
             ms * 1e3 / R / K);
    }
  return 0;
}
