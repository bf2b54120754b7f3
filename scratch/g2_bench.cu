// Standalone timing harness for the D = 256 gradient pass (development tool, not part of the
// library): netscale shapes (Na = Nb = 16384), synthetic statistics on the fast-factor path,
// ablation variants selected through Grad2Args::dbg.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2408_11052_b200/csrc \
//        scratch/g2_bench.cu build/obj/tc_gemm.o -o /tmp/g2_bench -lcuda && /tmp/g2_bench
#include "../paper_2408_11052_b200/csrc/tc_grad2.cu"
#include <cmath>
#include <random>
#include <vector>

namespace crl { namespace tc {
bool make_map_bf16(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
} }
using namespace crl;
using namespace crl::tc;

template <class T>
static T* up(const std::vector<T>& v) {
  T* p;
  cudaMalloc(&p, v.size() * sizeof(T));
  cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return p;
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 16384, D = 256, pad = 256;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::mt19937 gen(7);
  std::normal_distribution<float> nd(0.f, 0.3f);
  std::vector<__nv_bfloat16> hA[2];
  std::vector<float> hst[2];
  for (int s = 0; s < 2; ++s) {
    hA[s].resize((size_t)N * D);
    hst[s].assign(N + pad, 0.f);
    for (int i = 0; i < N; ++i) {
      float q = 0.f;
      for (int k = 0; k < D; ++k) {
        __nv_bfloat16 b = __float2bfloat16(nd(gen));
        hA[s][(size_t)i * D + k] = b;
        q += __bfloat162float(b) * __bfloat162float(b);
      }
      hst[s][i] = q;
    }
  }
  const float invN = 1.f / N, lse = 3.f;
  std::vector<float> lr(N + pad, lse), lcf(N + pad, std::exp2f(-lse * 1.4426950408889634f) * invN);
  __nv_bfloat16* dA0 = up(hA[0]);
  __nv_bfloat16* dA1 = up(hA[1]);
  float* st0 = up(hst[0]);
  float* st1 = up(hst[1]);
  float* dlr = up(lr);
  float* dlcf = up(lcf);
  std::vector<int> one(4, 1);
  int* fac = up(one);
  float *pda, *prs;
  cudaMalloc(&pda, (size_t)4 * N * D * 4);
  cudaMalloc(&prs, (size_t)16 * N * 4);
  CUtensorMap m0, m1;
  if (!make_map_bf16(&m0, dA1, D, N, D, 64, 128) || !make_map_bf16(&m1, dA0, D, N, D, 64, 128)) {
    printf("tensor map failed\n");
    return 1;
  }
  Grad2Args ga{};
  ga.Na = N; ga.Nb = N; ga.invN = invN; ga.fac_ok = fac;
  Grad2Side& s0 = ga.side[0];
  s0.a_stat = st0; s0.b_stat = st1; s0.lr = dlr; s0.lc = dlr; s0.lcf = dlcf;
  s0.c_r = 1.f; s0.c_c = 1.f; s0.beta_r = 0.1f; s0.beta_c = 0.f; s0.part_da = pda; s0.part_rs = prs; s0.A = dA0;
  Grad2Side& s1 = ga.side[1];
  s1 = s0;
  s1.a_stat = st1; s1.b_stat = st0; s1.beta_r = 0.f; s1.beta_c = 0.1f;
  s1.part_da = pda + (size_t)2 * N * D; s1.part_rs = prs + 4 * N; s1.A = dA1;
  const int grid = tc_grad2_grid(N, sms);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"full", "no-epi-math", "no-dA-mma", "", "no-S-mma", "", "S-only(no dA, no math)", "", "",
                         "", "", "", "", "", "", ""};
  const int variants[] = {0, 1};
  const double logits = 2.0 * N * (double)N, flops = 4.0 * N * (double)N * D * 2;
  for (int v : variants) {
    ga.dbg = v;
    for (int it = 0; it < 3; ++it) tc_grad2(CRL_ENERGY_L2, m0, m1, ga, grid, 0);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(err));
      return 1;
    }
    const int iters = 10;
    cudaEventRecord(e0);
    for (int it = 0; it < iters; ++it) tc_grad2(CRL_ENERGY_L2, m0, m1, ga, grid, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / iters;
    printf("dbg=%d %-26s %8.1f us  %7.1f TFLOP/s (4 GEMM-eq)  %6.2f Glogit-sides/ms\n", v,
           v < 16 && names[v][0] ? names[v] : "combo", us, flops / us * 1e-6, logits / us * 1e-6);
  }
  // ---- CTA-pair variant: time + compare slot sums of dA and row sums with the single-CTA pass
  {
    CUtensorMap s0m, s1m;
    if (!make_map_bf16(&s0m, dA1, D, N, D, 64, 64) || !make_map_bf16(&s1m, dA0, D, N, D, 64, 64)) {
      printf("tensor map failed\n");
      return 1;
    }
    ga.dbg = 0;
    const size_t nda = (size_t)4 * N * D, nrs = (size_t)16 * N;
    auto slot_sum = [&](std::vector<float>& da, std::vector<float>& rs, int nsub) {
      std::vector<float> h(nda), hr(nrs);
      cudaMemcpy(h.data(), pda, nda * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(hr.data(), prs, nrs * 4, cudaMemcpyDeviceToHost);
      da.assign((size_t)2 * N * D, 0.f);
      rs.assign((size_t)2 * N, 0.f);
      for (int sd = 0; sd < 2; ++sd)
        for (int sl = 0; sl < 2; ++sl)
          for (size_t i = 0; i < (size_t)N * D; ++i) da[sd * (size_t)N * D + i] += h[((size_t)sd * 2 + sl) * N * D + i];
      for (int sd = 0; sd < 2; ++sd)
        for (int u = 0; u < 2 * nsub; ++u)
          for (int i = 0; i < N; ++i) rs[sd * N + i] += hr[((size_t)sd * 2 * nsub + u) * N + i];
    };
    cudaMemset(pda, 0, nda * 4); cudaMemset(prs, 0, nrs * 4);
    tc_grad2(CRL_ENERGY_L2, m0, m1, ga, grid, 0);
    cudaDeviceSynchronize();
    std::vector<float> ref_da, ref_rs, got_da, got_rs;
    slot_sum(ref_da, ref_rs, 2);
    ga.side[1].part_rs = prs + (size_t)2 * 4 * N;         // pair: 4 warpgroup sub-slots per slot
    const int gp = tc_grad2p_grid(N, sms);
    cudaMemset(pda, 0, nda * 4); cudaMemset(prs, 0, nrs * 4);
    cudaError_t err = tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, ga, gp, 0);
    err = err != cudaSuccess ? err : cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("pair error %s\n", cudaGetErrorString(err)); return 1; }
    slot_sum(got_da, got_rs, 4);
    double md = 0, mr = 0, sd2 = 0, sr2 = 0;
    for (size_t i = 0; i < ref_da.size(); ++i) { md = std::max(md, (double)std::fabs(got_da[i] - ref_da[i])); sd2 = std::max(sd2, (double)std::fabs(ref_da[i])); }
    for (size_t i = 0; i < ref_rs.size(); ++i) { mr = std::max(mr, (double)std::fabs(got_rs[i] - ref_rs[i])); sr2 = std::max(sr2, (double)std::fabs(ref_rs[i])); }
    printf("pair vs single: max|d dA| %.3g (max %.3g)  max|d rs| %.3g (max %.3g)\n", md, sd2, mr, sr2);
    for (int it = 0; it < 3; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, ga, gp, 0);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, ga, gp, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / 10;
    printf("pair grid %d: %8.1f us  %7.1f TFLOP/s (4 GEMM-eq)\n", gp, us, flops / us * 1e-6);
    {
      setenv("CRL_G2P_V1", "1", 1);
      for (int it = 0; it < 3; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, ga, gp, 0);
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, ga, gp, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float m1s;
      cudaEventElapsedTime(&m1s, e0, e1);
      unsetenv("CRL_G2P_V1");
      printf("pair v1 (A in TMEM, one S buffer): %8.1f us\n", 1e3 * m1s / 10);
    }
    for (int v : {1, 2, 4, 3, 5, 6, 7}) {
      Grad2Args gv = ga;
      gv.dbg = v;
      for (int it = 0; it < 2; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, gv, gp, 0);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, gv, gp, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float m2;
      cudaEventElapsedTime(&m2, e0, e1);
      printf("  pair dbg=%d (%s%s%s): %8.1f us\n", v, v & 1 ? "no-math " : "", v & 2 ? "no-dA " : "", v & 4 ? "no-S" : "",
             1e3 * m2 / 5);
    }
    {
      unsigned long long* tr;
      cudaMalloc(&tr, 1024 * 8 * 8);
      cudaMemset(tr, 0, 1024 * 8 * 8);
      Grad2Args gt = ga;
      gt.trace = tr;
      tc_grad2p(CRL_ENERGY_L2, m0, m1, s0m, s1m, m1, m0, gt, gp, 0);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> ht(1024 * 8);
      cudaMemcpy(ht.data(), tr, ht.size() * 8, cudaMemcpyDeviceToHost);
      const unsigned long long t0 = ht[4];
      printf("pair trace: g: Sfree? Dfree Sissued dAissued Sready Sloaded mathdone Whanded\n");
      for (int g = 0; g < 24; ++g) {
        printf("%3d:", g);
        for (int e = 0; e < 8; ++e) printf(" %7lld", ht[g * 8 + e] ? (long long)(ht[g * 8 + e] - t0) : -1LL);
        printf("\n");
      }
      printf("pair period tiles 50..100: %.0f cyc/tile\n", (double)(ht[100 * 8 + 4] - ht[50 * 8 + 4]) / 50);
    }
  }
  // event trace of CTA 0 (full variant): per tile the clock of 0 B slot free, 1 S issued, 2 dA
  // issued, 3 S ready (epilogue), 4 S loaded, 5 math done, 6 W buffer free, 7 W handed over
  unsigned long long* tr;
  cudaMalloc(&tr, 1024 * 8 * 8);
  cudaMemset(tr, 0, 1024 * 8 * 8);
  ga.dbg = argc > 2 ? atoi(argv[2]) : 0;
  ga.trace = tr;
  tc_grad2(CRL_ENERGY_L2, m0, m1, ga, grid, 0);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> ht(1024 * 8);
  cudaMemcpy(ht.data(), tr, ht.size() * 8, cudaMemcpyDeviceToHost);
  const unsigned long long t0 = ht[4];
  printf("trace dbg=%d (cycles rel. to tile 0 S-ready):  g: B0free B1free Sissued dAissued Sready Sloaded mathdone Whanded\n", ga.dbg);
  for (int g = 0; g < 40; ++g) {
    printf("%3d:", g);
    for (int e = 0; e < 8; ++e) printf(" %7lld", ht[g * 8 + e] ? (long long)(ht[g * 8 + e] - t0) : -1LL);
    printf("\n");
  }
  for (int g = 50; g < 200; g += 50)
    printf("period tiles %d..%d: %.0f cyc/tile (S ready)\n", g, g + 50, (double)(ht[(g + 50) * 8 + 4] - ht[g * 8 + 4]) / 50);
  std::vector<float> h(8);
  cudaMemcpy(h.data(), pda, 32, cudaMemcpyDeviceToHost);
  printf("grid %d  sample dA %g %g\n", grid, h[0], h[1]);
  return 0;
}
