// tcgen05.mma issue-rate micro-benchmark (development tool, not part of the library):
// cycles per kind::f16 MMA (M = 128, K = 16, bf16 -> fp32) for N in {64, 128, 256}, with the A
// operand in SMEM (ss) or TMEM (ts), one CTA per SM, data left uninitialised (timing only).
// Also: LDTM (32x32b.x32) read throughput from 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2408_11052_b200/csrc \
//        scratch/mma_bench.cu -o scratch/mma_bench && scratch/mma_bench
#include <cstdio>
#include "tc_common.cuh"
#include "tc_pair.cuh"

using namespace crl::tc;

__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

constexpr int NMMA = 4096;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16_f32(128, N, false, false);
    const uint32_t a_base = smem_u32(smem), b_base = a_base + 65536;
    long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      const int ks = i & 3;
      const uint64_t bd = smem_desc_sw128(b_base + ks * 32, 16, 1024);
      if (TS) mma_ts(tmem, tmem + 256 + 8 * ks, bd, id, 1);
      else mma_bf16(tmem, smem_desc_sw128(a_base + ks * 32, 16, 1024), bd, id, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// the grad2 tile pattern: per tile S = A[tmem] . B^T (16 x N=64 K=16, A over 128 TMEM columns, B
// over 4 K-major SW128 chunks) into one of two 64-column buffers, then dA += W . B (4 x N=256,
// W K-major from SMEM, B MN-major).  MODE 1: S only, 2: dA only, 3: both.  INIT: random data
template <int MODE, bool INIT>
__global__ void __launch_bounds__(128, 1) k_tile(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, done_bar, dummy[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); mbar_init(&done_bar, 1);
    for (int i = 0; i < 3; ++i) mbar_init(&dummy[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  if (INIT) {
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < (32768 + 16384) / 4; i += blockDim.x) {
      uint32_t h = (uint32_t)i * 2654435761u;
      w[i] = (0x3c00u + (h & 0x3ffu)) | ((0x3c00u + ((h >> 10) & 0x3ffu)) << 16);   // bf16 ~ 1.x
      w[i] &= 0x3fff3fffu;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (INIT) {   // A (bf16 pairs) into TMEM columns 384..511
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = 0x3f803f80u ^ ((uint32_t)(lane + i) & 0x7fu);
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + 384 + 32 * c + ((uint32_t)(warp * 32) << 16)),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
          "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
          "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
          "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr int TILES = 256;
  if (MODE & 8) {
    // two issuing threads: warp 0 issues the S MMAs, warp 1 the dA MMAs, each with the
    // kernel-like control (waits on complete barriers, commits) between tiles
    if (threadIdx.x == 0) mbar_arrive(&done_bar);
    __syncthreads();
    if (lane == 0 && warp < 2) {
      const uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
      const uint32_t id_da = idesc_bf16_f32(128, 256, false, true);
      const uint32_t b_base = smem_u32(smem), w_base = b_base + 32768;
      long long t0 = clock64();
      for (int t = 0; t < TILES; ++t) {
        mbar_wait(&done_bar, 0); tc_fence_after();
        mbar_wait(&done_bar, 0); tc_fence_after();
        if (warp == 0) {
          for (int c = 0; c < 4; ++c)
            for (int ks = 0; ks < 4; ++ks)
              mma_ts(tmem + 64 * (t & 1), tmem + 384 + 8 * (4 * c + ks),
                     smem_desc_sw128(b_base + c * 8192 + ks * 32, 16, 1024), id_s, (c | ks) != 0);
          mma_commit(&dummy[0]);
        } else {
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(tmem + 128, smem_desc_sw128(w_base + ks * 32, 16, 1024),
                     smem_desc_sw128(b_base + ks * 2048, 8192, 1024), id_da, 1);
          mma_commit(&dummy[1]); mma_commit(&dummy[2]);
        }
      }
      if (warp == 0) {
        mma_commit(&bar);
        mbar_wait(&bar, 0);
      } else {
        mma_commit(&dummy[1]);
      }
      long long t1 = clock64();
      if (blockIdx.x == 0 && warp == 0) out[0] = (t1 - t0) / TILES;
    }
  } else if (threadIdx.x == 0) {
    const uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
    const uint32_t id_da = idesc_bf16_f32(128, 256, false, true);
    const uint32_t b_base = smem_u32(smem), w_base = b_base + 32768;
    long long t0 = clock64();
    if (MODE & 36) { mbar_arrive(&done_bar); }
    for (int t = 0; t < TILES; ++t) {
      if (MODE & 4) {   // the kernel's per-tile control: 2 waits on complete barriers, fences, commits
        mbar_wait(&done_bar, 0); tc_fence_after();
        mbar_wait(&done_bar, 0); tc_fence_after();
      }
      if (MODE & 32) { mbar_wait(&done_bar, 0); mbar_wait(&done_bar, 0); mbar_wait(&done_bar, 0); }
      if (MODE & 64) { tc_fence_after(); tc_fence_after(); tc_fence_after(); }
      if (MODE & 1)
        for (int c = 0; c < 4; ++c)
          for (int ks = 0; ks < 4; ++ks)
            mma_ts(tmem + 64 * (t & 1), tmem + 384 + 8 * (4 * c + ks), smem_desc_sw128(b_base + c * 8192 + ks * 32, 16, 1024),
                   id_s, (c | ks) != 0);
      if (MODE & 4) mma_commit(&dummy[0]);
      if (MODE & 4) { mbar_wait(&done_bar, 0); tc_fence_after(); }
      if (MODE & 2)
        for (int ks = 0; ks < 4; ++ks)
          mma_bf16(tmem + 128, smem_desc_sw128(w_base + ks * 32, 16, 1024), smem_desc_sw128(b_base + ks * 2048, 8192, 1024),
                   id_da, 1);
      if (MODE & 4) { mma_commit(&dummy[1]); mma_commit(&dummy[2]); }
      if (MODE & 16) { mma_commit(&dummy[0]); mma_commit(&dummy[1]); mma_commit(&dummy[2]); }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (t1 - t0) / TILES;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE, bool INIT>
void run_tile(int sms, long long* d) {
  const int smem = 65536;
  cudaFuncSetAttribute(k_tile<MODE, INIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k_tile<MODE, INIT><<<sms, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("tile mode %d (%s) init %d: %lld cyc/tile (floor S 512 + dA 512)  %s\n", MODE,
         MODE == 1 ? "S" : MODE == 2 ? "dA" : "S+dA", (int)INIT, c, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

// CTA-pair MMAs (cta_group::2, M = 256): cycles per instruction for N in {128, 256}, A from SMEM
// (ss) or TMEM (ts); the leader issues, completion multicast to both CTAs
template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_mma_pair(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = pair::cluster_rank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) pair::tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  pair::cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t id = idesc_bf16_f32(256, N, false, false);
    const uint32_t a_base = smem_u32(smem), b_base = a_base + 65536;
    long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      const int ks = i & 3;
      const uint64_t bd = smem_desc_sw128(b_base + ks * 32, 16, 1024);
      if (TS) pair::mma_pair_ts(tmem, tmem + 256 + 8 * ks, bd, id, 1);
      else pair::mma_pair(tmem, smem_desc_sw128(a_base + ks * 32, 16, 1024), bd, id, 1);
    }
    pair::commit_pair(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  pair::cluster_sync();
  if (warp == 0) { tc_fence_after(); pair::tmem_dealloc_pair(tmem, 512); }
}
template <int N, bool TS>
void run_mma_pair(int sms, long long* d) {
  const int smem = 65536 + 65536;
  cudaFuncSetAttribute(k_mma_pair<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k_mma_pair<N, TS><<<sms, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)c / NMMA;
  printf("pair mma %s N=%3d: %6.1f cyc/MMA  (floor %3d)  %s\n", TS ? "ts" : "ss", N, cyc, 256 * N / 512,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

// TMEM -> registers: every warp reads its 32 lanes x 32 columns, ITER times over 128 columns
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_ldtm(long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
    uint32_t r[32];
    tmem_ld32_nowait(tmem + lane_off + 32 * ((it + warp / 4) & 15), r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 1.2345f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run_mma(int sms, long long* d) {
  const int smem = 65536 + 65536;
  cudaFuncSetAttribute(k_mma<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k_mma<N, TS><<<sms, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)c / NMMA;
  printf("mma %s N=%3d: %6.1f cyc/MMA  (floor %3d)  %6.0f flop/cyc/SM  %s\n", TS ? "ts" : "ss", N, cyc, 128 * N / 256,
         2.0 * 128 * N * 16 / cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
template <int NW>
void run_ldtm(int sms, long long* d, float* s) {
  for (int rep = 0; rep < 2; ++rep) k_ldtm<NW><<<sms, NW * 32>>>(d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)NW * 1024 * 32 * 32 * 4;
  printf("ldtm %2d warps: %6.1f B/cyc/SM  %s\n", NW, bytes / c, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  run_mma<64, false>(sms, d);
  run_mma<64, true>(sms, d);
  run_mma<128, false>(sms, d);
  run_mma<128, true>(sms, d);
  run_mma<256, false>(sms, d);
  run_mma<256, true>(sms, d);
  run_mma_pair<128, false>(sms, d);
  run_mma_pair<128, true>(sms, d);
  run_mma_pair<256, false>(sms, d);
  run_mma_pair<256, true>(sms, d);
  run_tile<1, false>(sms, d);
  run_tile<2, false>(sms, d);
  run_tile<3, false>(sms, d);
  run_tile<7, false>(sms, d);
  run_tile<5, false>(sms, d);
  run_tile<4, false>(sms, d);
  run_tile<8, false>(sms, d);
  run_tile<16 + 3, false>(sms, d);
  run_tile<32 + 3, false>(sms, d);
  run_tile<64 + 3, false>(sms, d);
  run_ldtm<4>(sms, d, s);
  run_ldtm<8>(sms, d, s);
  run_ldtm<16>(sms, d, s);
  return 0;
}
