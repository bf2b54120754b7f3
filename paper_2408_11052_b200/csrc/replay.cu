// replay.cu — A0 buffer insert and A1 hindsight relabel sample (contract C1).
//
// Paper: Alg. 1 P:1030-1038 (per-env trajectories, reset on terminal), Table 2
// (capacity per env), §3 P:165-169 (goal T ~ Geom(1-gamma) steps ahead), §3.1 P:190-191 and
// §3.2 P:219 ((s,a) uniform, g from the states after s in the same trajectory), Alg. 1
// P:1045-1046 ("sample (with discount)").  Readings A-07..A-12, A-18.
//
// HBM layout (per rank, inside crl_memory.buffer):
//   obs_ring [E_l][T][obs_stride] fp32    act_ring [E_l][T][act_stride] fp32
//   ep_end   [E_l][T] u32  absolute index of the last slot of that slot's episode, or
//                          kOpen while the episode is still running
//   open_start [E_l] u32   absolute index where the currently open episode began
//   qtab     [T+1] u64     Q[k] = floor((1 - gamma^k) 2^64), built on the host
// Device index arithmetic is integer-only, so sampled indices are bit-exact.
#include <cmath>

#include "common.cuh"

namespace crl {

constexpr uint32_t kOpen = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11), counter (c0..c3), key (k0, k1)
// ---------------------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// ---------------------------------------------------------------------------------------
// A0: one CTA per env.  All threads copy the env's U new rows into the ring (coalesced
// per row), mark the new slots open, then warp 0 walks the U done flags and back-fills
// ep_end for every episode that closed (each slot is back-filled at most once).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) buffer_insert_kernel(
    const float* __restrict__ obs, const float* __restrict__ act, const uint8_t* __restrict__ done,
    int U, int E, int T, int obs_dim, int act_dim, int obs_stride, int act_stride,
    uint32_t n_ins, float* __restrict__ obs_ring, float* __restrict__ act_ring,
    uint32_t* __restrict__ ep_end, uint32_t* __restrict__ open_start) {
  const int e = blockIdx.x;
  const uint32_t n_new = n_ins + (uint32_t)U;
  // copy rows: a warp per step u (8 warps over the U steps), lanes along the row, every load
  // of a warp's rows issued before its stores (the rows are independent; one HBM latency per
  // group of 8 instead of one per row)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int RPW = 8;                                  // rows in flight per warp
  for (int u0 = warp; u0 < U; u0 += RPW * nw) {
    for (int c = lane; c < obs_dim; c += 32) {
      float v[RPW];
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int u = u0 + k * nw;
        v[k] = u < U ? obs[((size_t)u * E + e) * obs_dim + c] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int u = u0 + k * nw;
        if (u < U) obs_ring[((size_t)e * T + (n_ins + (uint32_t)u) % (uint32_t)T) * obs_stride + c] = v[k];
      }
    }
    for (int c = lane; c < act_dim; c += 32) {
      float v[RPW];
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int u = u0 + k * nw;
        v[k] = u < U ? act[((size_t)u * E + e) * act_dim + c] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int u = u0 + k * nw;
        if (u < U) act_ring[((size_t)e * T + (n_ins + (uint32_t)u) % (uint32_t)T) * act_stride + c] = v[k];
      }
    }
  }
  for (int u = threadIdx.x; u < U; u += blockDim.x) {
    uint32_t slot = (n_ins + u) % (uint32_t)T;
    ep_end[(size_t)e * T + slot] = kOpen;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  // episode ends: the U done flags are read 32 at a time (one ballot) and the closed episodes
  // are back-filled in step order (each slot at most once)
  uint32_t start = open_start[e];
  const uint32_t lo_keep = n_new > (uint32_t)T ? n_new - (uint32_t)T : 0u;   // oldest kept slot
  for (int u0 = 0; u0 < U; u0 += 32) {
    unsigned bits = __ballot_sync(0xffffffffu, u0 + lane < U && done[(size_t)(u0 + lane) * E + e] != 0);
    while (bits) {
      const int u = u0 + __ffs(bits) - 1;
      bits &= bits - 1u;
      const uint32_t tau_end = n_ins + (uint32_t)u;
      const uint32_t first = start > lo_keep ? start : lo_keep;
      for (uint32_t t = first + lane; t <= tau_end; t += 32)
        ep_end[(size_t)e * T + (t % (uint32_t)T)] = tau_end;
      start = tau_end + 1;
    }
  }
  if (lane == 0) open_start[e] = start;
}

// ---------------------------------------------------------------------------------------
// A1: a group of LPR lanes per row.  Lane a of the group evaluates attempt a (a + LPR, ...) of
// the rejection loop in parallel; the first accepted attempt (lowest a) wins via ballot, which reproduces the
// sequential "first valid attempt" of the contract.  The offset k is the inverse-CDF lookup
// k = min{k in [1, L] : Q[k] > t} in the u64 table Q (L2-resident): an fp64 estimate
// k~ = ceil(log(1 - t 2^-64) / log gamma) places a window of LPR entries around it (one load
// per lane), and a ballot over "Q[k] > t" takes the first index.  The decision is the
// exact integer comparison; the window is accepted only if it brackets the answer
// (Q[first - 1] <= t), else a binary search over Q in global memory decides (a fallback for
// estimates off by more than 16, which the fp64 estimate does not produce for T <= 2^20).
// Rows are then gathered by the group.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// LPR lanes per row (a warp holds 32 / LPR rows): LPR = 4 for the narrow rows of the paper's
// configs (more independent rows, i.e. gathers, in flight per warp), 32 for wide rows.
template <int LPR>
__global__ void __launch_bounds__(256) relabel_sample_kernel(
    int B_l, int n_upd, int rank, int E, int T, int obs_dim, int act_dim, int goal_dim, int goal_offset,
    int obs_stride, int act_stride, uint32_t tau_old, uint32_t tau_new,
    uint32_t seed_lo, uint32_t seed_hi, uint32_t step_lo0, uint32_t step_hi0, double log_gamma, uint64_t alpha_t,
    const float* __restrict__ obs_ring, const float* __restrict__ act_ring,
    const uint32_t* __restrict__ ep_end, const uint64_t* __restrict__ qtab,
    float* __restrict__ s_out, float* __restrict__ a_out, float* __restrict__ g_out,
    float* __restrict__ ga_out, int64_t* __restrict__ idx_out, int* __restrict__ status) {
  constexpr int RPW = 32 / LPR;                                 // rows per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int src0 = sub * LPR;                                   // first lane of this row's group
  // output row r = u B_l + rl: update u of a bulk call draws with step = step0 + u, exactly as
  // n_upd separate calls would (F4)
  const int r = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW + sub;
  if (r >= B_l * n_upd) return;                                 // uniform within the group
  const int u_upd = r / B_l, rl = r - u_upd * B_l;
  const uint64_t step64 = (((uint64_t)step_hi0 << 32) | step_lo0) + (uint64_t)u_upd;
  const uint32_t step_lo = (uint32_t)step64, step_hi = (uint32_t)(step64 >> 32);
  const uint32_t rho = (uint32_t)rank * (uint32_t)B_l + (uint32_t)rl;
  const uint32_t n = tau_new - tau_old + 1;

  // attempts a = base + li, LPR at a time; the first accepted one (lowest a) wins
  int found = -1;
  uint32_t e = 0, tau = 0, L = 0, x2 = 0, x3 = 0;
  for (int base = 0; base < 64 && found < 0; base += LPR) {
    const uint32_t att = (uint32_t)(base + li);
    U4 x = philox4x32_10(U4{rho, att, step_lo, step_hi}, seed_lo, seed_hi);
    uint32_t ee = (uint32_t)(((uint64_t)x.x * (uint64_t)E) >> 32);
    uint32_t j = (uint32_t)(((uint64_t)x.y * (uint64_t)n) >> 32);
    uint32_t t = tau_old + j;
    uint32_t end = ep_end[(size_t)ee * T + (t % (uint32_t)T)];
    uint32_t cap = end < tau_new ? end : tau_new;          // kOpen > tau_new always
    uint32_t LL = cap - t;
    const unsigned ok = (__ballot_sync(gmask, LL >= 1u) & gmask) >> src0;
    if (ok) {
      const int src = src0 + __ffs(ok) - 1;
      found = base + __ffs(ok) - 1;
      e = __shfl_sync(gmask, ee, src);
      tau = __shfl_sync(gmask, t, src);
      L = __shfl_sync(gmask, LL, src);
      x2 = __shfl_sync(gmask, x.z, src);
      x3 = __shfl_sync(gmask, x.w, src);
    }
  }
  if (found < 0) {
    if (li == 0) set_status(status, CRL_ESAMPLER);
    // deterministic fill so downstream stays finite
    e = 0; tau = tau_old; L = 1; x2 = 0; x3 = 0;
  }
  // k = min{k in [1, L] : Q[k] > t},  t = (R * Q[L]) >> 64   (Q[0] = 0 <= t < Q[L])
  const uint64_t R = ((uint64_t)x2 << 32) | (uint64_t)x3;
  const uint64_t tt = mulhi64(R, __ldg(qtab + L));
  const double u = (double)tt * 5.421010862427522e-20;          // t 2^-64
  const double kf = ceil(log1p(-u) / log_gamma);
  const uint32_t kest = kf >= 1.0 ? (kf <= (double)L ? (uint32_t)kf : L) : 1u;
  constexpr uint32_t kBack = LPR / 4;                           // window Q[base-1 .. base+LPR-2]
  const uint32_t wbase = kest > kBack ? kest - kBack : 1u;
  const uint32_t kw = wbase - 1u + (uint32_t)li;
  const bool above = kw > L || __ldg(qtab + kw) > tt;
  const unsigned bal = (__ballot_sync(gmask, above) & gmask) >> src0;
  uint32_t k;
  if (bal != 0u && (bal & 1u) == 0u) {
    k = wbase - 1u + (uint32_t)(__ffs(bal) - 1);
  } else {
    uint32_t lo = 1, hi = L;                   // invariant: answer in [lo, hi], Q[hi] > tt
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(qtab + mid) > tt) hi = mid; else lo = mid + 1;
    }
    k = lo;
  }
  const uint32_t slot = tau % (uint32_t)T;
  const uint32_t gslot = (tau + k) % (uint32_t)T;
  const float* srow = obs_ring + ((size_t)e * T + slot) * obs_stride;
  const float* arow = act_ring + ((size_t)e * T + slot) * act_stride;
  const float* grow = obs_ring + ((size_t)e * T + gslot) * obs_stride + goal_offset;
  float* so = s_out + (size_t)r * obs_dim;
  float* ao = a_out + (size_t)r * act_dim;
  float* go = g_out + (size_t)r * goal_dim;
  for (int c = li; c < obs_dim; c += LPR) so[c] = srow[c];
  for (int c = li; c < act_dim; c += LPR) ao[c] = arow[c];
  for (int c = li; c < goal_dim; c += LPR) go[c] = grow[c];
  if (ga_out != nullptr) {
    // the ACTOR's goals with random-goal mixing (F4, App. C P:951-964 mixes random goals into
    // the policy objective only, reading A-36): draw 64 (past the start attempts) decides
    // and places it; the critic's g above stays the hindsight goal
    const float* garow = grow;
    if (alpha_t != 0) {
      const U4 y = philox4x32_10(U4{rho, 64u, step_lo, step_hi}, seed_lo, seed_hi);
      if ((uint64_t)y.x < alpha_t) {
        const uint32_t ge = (uint32_t)(((uint64_t)y.y * (uint64_t)E) >> 32);
        const uint32_t gs = (tau_old + (uint32_t)(((uint64_t)y.z * (uint64_t)n) >> 32)) % (uint32_t)T;
        garow = obs_ring + ((size_t)ge * T + gs) * obs_stride + goal_offset;
      }
    }
    float* gao = ga_out + (size_t)r * goal_dim;
    for (int c = li; c < goal_dim; c += LPR) gao[c] = garow[c];
  }
  if (idx_out != nullptr && li < 3) {
    int64_t v = li == 0 ? (int64_t)rank * E + e : (li == 1 ? (int64_t)tau : (int64_t)(tau + k));
    idx_out[(size_t)r * 3 + li] = v;
  }
}

// ---------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------
cudaError_t launch_buffer_insert(const float* obs, const float* act, const uint8_t* done, int U,
                                 int E, int T, int obs_dim, int act_dim, int obs_stride,
                                 int act_stride, uint32_t n_ins, float* obs_ring, float* act_ring,
                                 uint32_t* ep_end, uint32_t* open_start, cudaStream_t st) {
  buffer_insert_kernel<<<E, 256, 0, st>>>(obs, act, done, U, E, T, obs_dim, act_dim, obs_stride,
                                          act_stride, n_ins, obs_ring, act_ring, ep_end, open_start);
  return cudaGetLastError();
}

cudaError_t launch_relabel_sample(int B_l, int n_upd, int rank, int E, int T, int obs_dim, int act_dim,
                                  int goal_dim, int goal_offset, int obs_stride, int act_stride,
                                  uint32_t tau_old, uint32_t tau_new, uint64_t seed, uint64_t step, double gamma,
                                  uint64_t alpha_t,
                                  const float* obs_ring, const float* act_ring,
                                  const uint32_t* ep_end, const uint64_t* qtab, float* s, float* a,
                                  float* g, float* g_actor, int64_t* idx, int* status, cudaStream_t st) {
  const int warps = 8;
  const long rows = (long)B_l * n_upd;
  // narrow rows (the paper's Reacher / Ant; Humanoid is wide) in large batches: 8 rows per warp
  // for memory-level parallelism; small batches keep a warp per row (latency: measured at
  // Ant B = 256, 10.3 us vs 12.3 us with 8 rows per warp)
  const bool narrow = obs_dim <= 64 && rows >= 8192;
  const int rpw = narrow ? 8 : 1;
  dim3 grid((unsigned)((rows + (long)warps * rpw - 1) / ((long)warps * rpw)));
  auto kern = narrow ? relabel_sample_kernel<4> : relabel_sample_kernel<32>;
  kern<<<grid, warps * 32, 0, st>>>(
      B_l, n_upd, rank, E, T, obs_dim, act_dim, goal_dim, goal_offset, obs_stride, act_stride, tau_old,
      tau_new, (uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)step, (uint32_t)(step >> 32), std::log(gamma), alpha_t,
      obs_ring, act_ring, ep_end, qtab, s, a, g, g_actor, idx, status);
  return cudaGetLastError();
}

}  // namespace crl
