// Throughput of the SFU (MUFU) and packed-FMA instruction mixes on this GPU, in lane-ops per
// clock per SM.  Calibration for the XU roofline of tc_stats / tc_gradf.  Not part of the library.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

constexpr int ITERS = 4096, CH = 8;

template <int OP>
__global__ void k(float* out, long long* cyc) {
  float x[CH];
  unsigned h[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = 0.1f + 0.01f * (threadIdx.x + c); h[c] = 0x3c003c00u + c; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(x[c]) : "f"(-x[c]));
      if (OP == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(x[c]) : "f"(x[c]));
      if (OP == 2) asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(x[c]) : "f"(x[c]));
      if (OP == 3) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(h[c]) : "r"(h[c] ^ 0x80008000u));
      if (OP == 4) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(h[c]) : "r"(h[c] ^ 0x80008000u));
      if (OP == 5) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(x[c]) : "f"(x[c]));
      if (OP == 6) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(x[c]) : "f"(x[c]));
      if (OP == 7) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(x[c]) : "f"(x[c]));
      if (OP == 8) {   // packed FFMA2 (counts 2 lane-ops per lane)
        unsigned long long v = ((unsigned long long)__float_as_uint(x[c]) << 32) | __float_as_uint(x[c]);
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
        x[c] = __uint_as_float((unsigned)v);
      }
      if (OP == 9) asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(h[c]) : "r"(h[c]));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + __uint_as_float(h[c]);
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_lane) {
  float* out; long long* cyc; long long hc;
  cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps = 8; warps <= 32; warps *= 2) {
    k<OP><<<sms, warps * 32>>>(out, cyc);
    cudaDeviceSynchronize();
    k<OP><<<sms, warps * 32>>>(out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (double)warps * 32 * ITERS * CH * per_lane;
    printf("%-22s warps/SM=%2d  %.2f lane-ops/clk/SM\n", name, warps, ops / hc);
  }
}

int main() {
  run<0>("ex2.f32", 1);
  run<1>("rsqrt.f32", 1);
  run<2>("sqrt.f32", 1);
  run<3>("ex2.f16x2", 2);
  run<4>("ex2.bf16x2", 2);
  run<5>("tanh.f32", 1);
  run<6>("rcp.f32", 1);
  run<7>("lg2.f32", 1);
  run<8>("fma.f32x2", 2);
  run<9>("tanh.f16x2", 2);
  return 0;
}
