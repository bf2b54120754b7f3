// Standalone correctness + timing harness for tc_pgemm (development tool, not part of the library):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2408_11052_b200/csrc \
//        scratch/pgemm_test.cu -o /tmp/pgemm_test -lcuda && /tmp/pgemm_test
#include "../paper_2408_11052_b200/csrc/tc_gemm.cu"
#include "../paper_2408_11052_b200/csrc/tc_pgemm.cu"
#include <vector>
#include <cmath>
#include <random>

using namespace crl;
using namespace crl::tc;

__global__ void ref_gemm(const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, int M, int N, int K, bool b_kn,
                         float* C) {
  // C[m][n] = sum_k A[m][k] * (b_kn ? B[k][n] : B[n][k])
  int m = blockIdx.y * 16 + threadIdx.y, n = blockIdx.x * 16 + threadIdx.x;
  if (m >= M || n >= N) return;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) {
    float a = __bfloat162float(A[(size_t)m * lda + k]);
    float b = b_kn ? __bfloat162float(B[(size_t)k * N + n]) : __bfloat162float(B[(size_t)n * K + k]);
    acc += a * b;
  }
  C[(size_t)m * N + n] = acc;
}

static std::vector<__nv_bfloat16> rnd_bf16(size_t n, float sc, int seed) {
  std::mt19937 g(seed);
  std::normal_distribution<float> d(0.f, sc);
  std::vector<__nv_bfloat16> v(n);
  for (auto& x : v) x = __float2bfloat16(d(g));
  return v;
}
template <class T>
static T* up(const std::vector<T>& v) {
  T* p;
  cudaMalloc(&p, v.size() * sizeof(T));
  cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return p;
}
static std::vector<float> bf2f(const __nv_bfloat16* d, size_t n) {
  std::vector<__nv_bfloat16> h(n);
  cudaMemcpy(h.data(), d, n * 2, cudaMemcpyDeviceToHost);
  std::vector<float> f(n);
  for (size_t i = 0; i < n; ++i) f[i] = __bfloat162float(h[i]);
  return f;
}
static float silu(float z) { return z / (1.f + std::exp(-z)); }
static float silu_g(float z) { float s = 1.f / (1.f + std::exp(-z)); return s * (1.f + z * (1.f - s)); }

int main(int argc, char** argv) {
  int M = argc > 1 ? atoi(argv[1]) : 16384, N = argc > 2 ? atoi(argv[2]) : 1024, K = argc > 3 ? atoi(argv[3]) : 1024;
  setvbuf(stdout, nullptr, _IONBF, 0);
  int lda = (K + 7) / 8 * 8;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("M=%d N=%d K=%d sms=%d smem=%zu\n", M, N, K, sms, pg::kSmem);
  auto hX = rnd_bf16((size_t)M * lda, 1.f, 1);
  for (int m = 0; m < M; ++m) for (int k = K; k < lda; ++k) hX[(size_t)m * lda + k] = __float2bfloat16(0.f);
  auto hW = rnd_bf16((size_t)K * N, 1.f / std::sqrt((float)K), 2);
  std::vector<float> hb(N);
  for (int i = 0; i < N; ++i) hb[i] = 0.01f * (i % 17) - 0.08f;
  __nv_bfloat16 *X = up(hX), *W = up(hW);
  float* bias = up(hb);
  __nv_bfloat16 *Z, *Xn;
  cudaMalloc(&Z, (size_t)M * N * 2);
  cudaMalloc(&Xn, (size_t)M * N * 2);
  float* C;
  cudaMalloc(&C, (size_t)M * N * 4);
  // ---- forward hidden
  PgemmMaps mp{};
  bool ok = make_map_bf16(&mp.a, X, K, M, lda, 64, 128) && make_map_bf16(&mp.b, W, N, K, N, 64, 64) &&
            make_map_bf16(&mp.out0, Z, N, M, N, 64, 32) && make_map_bf16(&mp.out1, Xn, N, M, N, 64, 32);
  if (!ok) { printf("map fail\n"); return 1; }
  PgemmArgs pa{M, N, K, bias, CRL_ACT_SILU, nullptr, 0};
  cudaError_t e = tc_pgemm(PG_FWD_HIDDEN, mp, pa, sms, 0);
  e = e != cudaSuccess ? e : cudaDeviceSynchronize();
  printf("fwd launch: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  ref_gemm<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(X, lda, W, M, N, K, true, C);
  cudaDeviceSynchronize();
  std::vector<float> hC((size_t)M * N);
  cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
  auto gz = bf2f(Z, (size_t)M * N), gx = bf2f(Xn, (size_t)M * N);
  double mz = 0, mx = 0, ref = 0;
  for (size_t i = 0; i < hC.size(); ++i) {
    float z = hC[i] + hb[i % N];
    mz = std::max(mz, (double)std::fabs(gz[i] - z));
    mx = std::max(mx, (double)std::fabs(gx[i] - silu(z)));
    ref = std::max(ref, (double)std::fabs(z));
  }
  printf("fwd hidden: max|dZ| %.4g  max|dX| %.4g  (max|Z| %.3g)\n", mz, mx, ref);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) tc_pgemm(PG_FWD_HIDDEN, mp, pa, sms, 0);
  cudaEventRecord(e0);
  const int IT = 50;
  for (int i = 0; i < IT; ++i) tc_pgemm(PG_FWD_HIDDEN, mp, pa, sms, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double us = ms * 1e3 / IT;
  printf("fwd hidden: %.2f us  %.1f TFLOP/s\n", us, 2.0 * M * N * K / (us * 1e-6) / 1e12);
  if (argc > 4) {                          // quick mode (ncu): one more launch with dbg = argv[4]
    PgemmArgs px = pa;
    px.dbg = atoi(argv[4]);
    tc_pgemm(PG_FWD_HIDDEN, mp, px, sms, 0);
    cudaDeviceSynchronize();
    return 0;
  }
  // ablations (PgemmArgs::dbg): 1 no epilogue, 2 no MMA, 4 no TMA operand traffic
  for (int dbg : {1, 2, 4, 3, 5, 6, 7, 8, 16, 24, 10, 18, 26, 14, 30}) {
    PgemmArgs px = pa;
    px.dbg = dbg;
    for (int i = 0; i < 3; ++i) tc_pgemm(PG_FWD_HIDDEN, mp, px, sms, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < IT; ++i) tc_pgemm(PG_FWD_HIDDEN, mp, px, sms, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double u2 = ms * 1e3 / IT;
    printf("  dbg=%2d (%s%s%s%s%s): %.2f us  %.1f TFLOP/s-equiv\n", dbg, dbg & 1 ? "no-epi " : "", dbg & 2 ? "no-mma " : "",
           dbg & 4 ? "no-tma " : "", dbg & 8 ? "no-store " : "", dbg & 16 ? "no-act" : "", u2,
           2.0 * M * N * K / (u2 * 1e-6) / 1e12);
  }
  {
    long long* tr;
    cudaMalloc(&tr, 1024 * 8);
    cudaMemset(tr, 0, 1024 * 8);
    PgemmArgs px = pa;
    px.trace = tr;
    for (int dbg : {0, 2}) {
      px.dbg = dbg;
      tc_pgemm(PG_FWD_HIDDEN, mp, px, sms, 0);
      cudaDeviceSynchronize();
      std::vector<long long> h(1024);
      cudaMemcpy(h.data(), tr, 1024 * 8, cudaMemcpyDeviceToHost);
      {
        long long s0 = h[512], e1 = 0;
        for (int c = 0; c < 74; ++c) { s0 = std::min(s0, h[512 + 2 * c]); e1 = std::max(e1, h[513 + 2 * c]); }
        printf("cluster spans (ns from first start): ");
        for (int c = 0; c < 74; c += 1) printf("%d:%lld-%lld ", c, h[512 + 2 * c] - s0, h[513 + 2 * c] - s0);
        printf("\n  first start -> last end %lld ns\n", e1 - s0);
      }
      const long long t0 = h[264];
      printf("trace dbg=%d (cycles from tile 0 epilogue start): tile: mma-commit epi-start | chunk c: ld-done wait-done sts-done\n", dbg);
      for (int it = 0; it < 4; ++it) {
        printf("  tile %d: %8lld %8lld |", it, h[256 + it] - t0, h[264 + it] - t0);
        for (int c = 0; c < 4; ++c)
          printf(" [%lld %lld %lld]", h[(it * 4 + c) * 4] - t0, h[(it * 4 + c) * 4 + 1] - t0, h[(it * 4 + c) * 4 + 2] - t0);
        printf("\n");
      }
    }
  }
  // ---- dX: A = dZ [M][K2], W [N][K2] (in = N, out = K2)
  {
    const int K2 = N, N2 = K;          // dX of this layer: out = N, in = K
    if (N2 % 64 == 0 && N2 >= 256) {
      auto hdz = rnd_bf16((size_t)M * K2, 1.f, 3);
      auto hzp = rnd_bf16((size_t)M * N2, 1.f, 4);
      __nv_bfloat16 *dz = up(hdz), *zp = up(hzp), *out;
      cudaMalloc(&out, (size_t)M * N2 * 2);
      PgemmMaps md{};
      ok = make_map_bf16(&md.a, dz, K2, M, K2, 64, 128) && make_map_bf16(&md.b, W, K2, N2, K2, 64, 128) &&
           make_map_bf16(&md.out0, out, N2, M, N2, 64, 32) && make_map_bf16(&md.zin, zp, N2, M, N2, 64, 32);
      PgemmArgs pd{M, N2, K2, nullptr, CRL_ACT_SILU, nullptr, 0};
      e = tc_pgemm(PG_DX, md, pd, sms, 0);
      e = e != cudaSuccess ? e : cudaDeviceSynchronize();
      printf("dx launch: %s\n", cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      float* C2;
      cudaMalloc(&C2, (size_t)M * N2 * 4);
      // W stored [K][N] = [in][out]: as B K-major {K2=out, N2=in}: B[n][k] = W[n * N + k]
      ref_gemm<<<dim3((N2 + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(dz, K2, W, M, N2, K2, false, C2);
      cudaDeviceSynchronize();
      std::vector<float> hC2((size_t)M * N2);
      cudaMemcpy(hC2.data(), C2, hC2.size() * 4, cudaMemcpyDeviceToHost);
      auto go = bf2f(out, (size_t)M * N2);
      double md_ = 0, rf = 0;
      for (size_t i = 0; i < hC2.size(); ++i) {
        float r = hC2[i] * silu_g(__bfloat162float(hzp[i]));
        md_ = std::max(md_, (double)std::fabs(go[i] - r));
        rf = std::max(rf, (double)std::fabs(r));
      }
      printf("dx: max|err| %.4g (max|ref| %.3g)\n", md_, rf);
      for (int i = 0; i < 3; ++i) tc_pgemm(PG_DX, md, pd, sms, 0);
      cudaEventRecord(e0);
      for (int i = 0; i < IT; ++i) tc_pgemm(PG_DX, md, pd, sms, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      us = ms * 1e3 / IT;
      printf("dx: %.2f us  %.1f TFLOP/s\n", us, 2.0 * M * N2 * K2 / (us * 1e-6) / 1e12);
    }
  }
  // ---- output layer: N = 256
  {
    const int N3 = 256;
    auto hW3 = rnd_bf16((size_t)K * N3, 1.f / std::sqrt((float)K), 5);
    __nv_bfloat16* W3 = up(hW3);
    std::vector<float> hb3(N3, 0.05f);
    float* b3 = up(hb3);
    float *Y, *stat;
    __nv_bfloat16* Yb;
    cudaMalloc(&Y, (size_t)M * N3 * 4);
    cudaMalloc(&Yb, (size_t)M * N3 * 2);
    cudaMalloc(&stat, (size_t)M * 4);
    PgemmMaps mo{};
    ok = make_map_bf16(&mo.a, X, K, M, lda, 64, 128) && make_map_bf16(&mo.b, W3, N3, K, N3, 64, 64) &&
         make_map_f32(&mo.out0, Y, N3, M, N3, 32, 32) && make_map_bf16(&mo.out1, Yb, N3, M, N3, 64, 32);
    PgemmArgs po{M, N3, K, b3, CRL_ACT_SILU, stat, CRL_ENERGY_L2};
    e = tc_pgemm(PG_FWD_OUT, mo, po, sms, 0);
    e = e != cudaSuccess ? e : cudaDeviceSynchronize();
    printf("out launch: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float* C3;
    cudaMalloc(&C3, (size_t)M * N3 * 4);
    ref_gemm<<<dim3((N3 + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(X, lda, W3, M, N3, K, true, C3);
    cudaDeviceSynchronize();
    std::vector<float> r((size_t)M * N3), gy((size_t)M * N3), gs(M);
    cudaMemcpy(r.data(), C3, r.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(gy.data(), Y, gy.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(gs.data(), stat, M * 4, cudaMemcpyDeviceToHost);
    auto gyb = bf2f(Yb, (size_t)M * N3);
    double my = 0, myb = 0, ms_ = 0, rf = 0;
    for (int m = 0; m < M; ++m) {
      double sq = 0;
      for (int n = 0; n < N3; ++n) {
        size_t i = (size_t)m * N3 + n;
        float y = r[i] + 0.05f;
        my = std::max(my, (double)std::fabs(gy[i] - y));
        myb = std::max(myb, (double)std::fabs(gyb[i] - y));
        rf = std::max(rf, (double)std::fabs(y));
        sq += (double)gyb[i] * gyb[i];
      }
      ms_ = std::max(ms_, std::fabs(sq - gs[m]) / std::max(1.0, sq));
    }
    printf("out: max|dY32| %.4g max|dYbf| %.4g stat rel %.3g (max|Y| %.3g)\n", my, myb, ms_, rf);
    for (int i = 0; i < 3; ++i) tc_pgemm(PG_FWD_OUT, mo, po, sms, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < IT; ++i) tc_pgemm(PG_FWD_OUT, mo, po, sms, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    us = ms * 1e3 / IT;
    printf("out: %.2f us  %.1f TFLOP/s\n", us, 2.0 * M * N3 * K / (us * 1e-6) / 1e12);
  }
  return 0;
}
