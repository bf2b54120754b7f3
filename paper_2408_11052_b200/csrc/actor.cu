// actor.cu — crl_actor_loss: the CRL actor objective with the critic frozen (fp32 SIMT).
//
// Paper: Eq. 3 P:212-218 (max_pi E[f(phi(s, a'), psi(g))], a' ~ pi(.|s, g)), the tunable
// entropy coefficient, SAC-style tanh-Gaussian policy (App. C; readings A-26/A-27:
// log sigma clipped to [-5, 2], gradient 0 outside; log pi with the tanh correction
// log(1 - a'^2 + 1e-6)).  Oracle: oracle/critic.py actor_loss.
//
//   [mu, log sigma_raw] = pi([s || g])                       (actor MLP, SiLU/ReLU hidden)
//   u = mu + sigma eps, a' = tanh(u)                           (eps ~ N(0, 1) is an input)
//   log pi = sum_k (-eps_k^2/2 - log sigma_k - log(2 pi)/2 - log(1 - a'_k^2 + 1e-6))
//   L = (1/N) sum_i (alpha log pi_i - f(phi([s_i || a'_i]), psi(g_i)))   (global mean)
// Reverse mode: dPhi_i = -(1/N) df/dphi_i -> phi's dX chain (dX only, critic frozen) ->
// dL/da' = the action columns of dX_0 -> head VJP -> actor backward (dW, db, dX) -> optional
// all-reduce (DP) -> optional Adam step (lr_actor) on the actor parameters.
//
// The step is small (a few GEMMs at width 256) and runs eagerly on `stream`; the GEMMs are
// the fp32 SIMT kernels of mlp_simt.cu, the per-row head / energy kernels below.
#include <cmath>

#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace crl {

constexpr float kLogSigMin = -5.f, kLogSigMax = 2.f;
constexpr float kHalfLog2Pi = 0.91893853320467274178f;   // log(2 pi) / 2

// 1 - tanh(u)^2 = sech(u)^2, evaluated without the cancellation of 1 - a'^2 in fp32 when
// |a'| -> 1 (the oracle's fp64 1 - a'^2 is exact enough; fp32 is not)
__device__ __forceinline__ float one_minus_tanh2(float u) {
  const float c = coshf(u);
  return 1.f / (c * c);
}

// per row: a' and log pi from the actor output and the noise
__global__ void actor_head_fwd_kernel(int Bl, int A, const float* __restrict__ out, const float* __restrict__ eps,
                                      float* __restrict__ a_new, float* __restrict__ logpi) {
  pdl_wait();
  pdl_launch();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= Bl) return;
  float lp = 0.f;
  for (int k = 0; k < A; ++k) {
    const float mu = out[(size_t)row * 2 * A + k];
    const float ls = fminf(fmaxf(out[(size_t)row * 2 * A + A + k], kLogSigMin), kLogSigMax);
    const float e = eps[(size_t)row * A + k];
    const float u = fmaf(expf(ls), e, mu);
    a_new[(size_t)row * A + k] = tanhf(u);
    lp += -0.5f * e * e - ls - kHalfLog2Pi - logf(one_minus_tanh2(u) + 1e-6f);
  }
  logpi[row] = lp;
}

// one warp per row: f_i = f(phi_i, psi_i), dPhi_i = -(1/N) df/dphi_i, rowloss_i = alpha log pi_i - f_i
__global__ void actor_diag_kernel(int Bl, int D, int energy, float invN, const float* __restrict__ alpha_p,
                                  const float* __restrict__ phi,
                                  const float* __restrict__ psi, const float* __restrict__ logpi,
                                  float* __restrict__ dphi, float* __restrict__ rowloss) {
  pdl_wait();
  pdl_launch();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= Bl) return;
  const float* x = phi + (size_t)row * D;
  const float* y = psi + (size_t)row * D;
  float* dx = dphi + (size_t)row * D;
  float f;
  if (energy == CRL_ENERGY_L2) {                 // f = -sqrt(|x - y|^2 + eps2)
    float ss = 0.f;
    for (int k = lane; k < D; k += 32) { const float d = x[k] - y[k]; ss = fmaf(d, d, ss); }
    ss = warp_sum(ss);
    const float r = sqrtf(ss + kEpsL2);
    f = -r;
    const float c = invN / r;                    // -(1/N) * (-(x - y) / r)
    for (int k = lane; k < D; k += 32) dx[k] = c * (x[k] - y[k]);
  } else if (energy == CRL_ENERGY_L2SQ) {        // f = -|x - y|^2, df/dx = -2 (x - y)
    float ss = 0.f;
    for (int k = lane; k < D; k += 32) { const float d = x[k] - y[k]; ss = fmaf(d, d, ss); }
    f = -warp_sum(ss);
    for (int k = lane; k < D; k += 32) dx[k] = 2.f * invN * (x[k] - y[k]);
  } else if (energy == CRL_ENERGY_L1) {          // f = -|x - y|_1, df/dx = -sign(x - y)
    float sa = 0.f;
    for (int k = lane; k < D; k += 32) sa += fabsf(x[k] - y[k]);
    f = -warp_sum(sa);
    for (int k = lane; k < D; k += 32) {
      const float d = x[k] - y[k];
      dx[k] = invN * (float)((d > 0.f) - (d < 0.f));
    }
  } else if (energy == CRL_ENERGY_DOT) {         // f = x . y
    float s = 0.f;
    for (int k = lane; k < D; k += 32) s = fmaf(x[k], y[k], s);
    f = warp_sum(s);
    for (int k = lane; k < D; k += 32) dx[k] = -invN * y[k];
  } else {                                       // f = x . y / (max(|x|, e) max(|y|, e))
    float xx = 0.f, yy = 0.f, xy = 0.f;
    for (int k = lane; k < D; k += 32) {
      xx = fmaf(x[k], x[k], xx); yy = fmaf(y[k], y[k], yy); xy = fmaf(x[k], y[k], xy);
    }
    xx = warp_sum(xx); yy = warp_sum(yy); xy = warp_sum(xy);
    const float nxr = sqrtf(xx), nyr = sqrtf(yy);
    const float nx = fmaxf(nxr, kEpsCos), ny = fmaxf(nyr, kEpsCos);
    f = xy / nx / ny;
    // df/dx = (v - (v.u) u) / nx with v = y / ny, u = x / nx  (|x| > eps), else v / eps
    const float proj = xy / (nx * ny);           // v . u
    for (int k = lane; k < D; k += 32) {
      const float v = y[k] / ny;
      const float g = nxr > kEpsCos ? (v - proj * (x[k] / nx)) / nx : v / kEpsCos;
      dx[k] = -invN * g;
    }
  }
  if (lane == 0) rowloss[row] = *alpha_p * logpi[row] - f;
}

// one CTA: deterministic sums of the per-row losses and log pi into a_loss[0..1]
__global__ void __launch_bounds__(1024) actor_loss_sum_kernel(int Bl, const float* __restrict__ rowloss,
                                                              const float* __restrict__ logpi,
                                                              float* __restrict__ acc) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[2][32];
  float s = 0.f, lp = 0.f;
  for (int i = threadIdx.x; i < Bl; i += blockDim.x) { s += rowloss[i]; lp += logpi[i]; }
  s = warp_sum(s);
  lp = warp_sum(lp);
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s; red[1][threadIdx.x >> 5] = lp; }
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[0][threadIdx.x] : 0.f;
    float w = threadIdx.x < (blockDim.x >> 5) ? red[1][threadIdx.x] : 0.f;
    v = warp_sum(v);
    w = warp_sum(w);
    if (threadIdx.x == 0) { acc[0] = v; acc[1] = w; }
  }
}

// loss = acc / N; non-finite -> skip the actor Adam step and raise the status word
__global__ void actor_loss_finalize_kernel(float* __restrict__ acc, float invN, float* __restrict__ loss_out,
                                           int* __restrict__ skip, int* __restrict__ t, int apply_adam,
                                           int* __restrict__ status) {
  pdl_wait();
  pdl_launch();
  const float L = acc[0] * invN;
  acc[2] = L;
  acc[3] = acc[1] * invN;                          // mean log pi (global): the entropy update's input
  if (loss_out) loss_out[0] = L;
  const bool bad = !isfinite(L);
  if (bad) set_status(status, CRL_ENONFINITE);
  *skip = (bad || !apply_adam) ? 1 : 0;
  if (!bad && apply_adam) *t += 1;
}

// per row: dL/d(mu, log sigma_raw) from dL/da' (critic path) and the log pi terms
__global__ void actor_head_bwd_kernel(int Bl, int A, const float* __restrict__ alpha_p, float invN,
                                      const float* __restrict__ out,
                                      const float* __restrict__ eps, const float* __restrict__ a_new,
                                      const float* __restrict__ da, float* __restrict__ dout) {
  const float alpha_invN = *alpha_p * invN;
  pdl_wait();
  pdl_launch();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= Bl) return;
  for (int k = 0; k < A; ++k) {
    const float an = a_new[(size_t)row * A + k];
    const float lsr = out[(size_t)row * 2 * A + A + k];
    const float ls = fminf(fmaxf(lsr, kLogSigMin), kLogSigMax);
    const float sig = expf(ls), e = eps[(size_t)row * A + k];
    const float one_m = one_minus_tanh2(fmaf(sig, e, out[(size_t)row * 2 * A + k]));
    // d/du of [f-term through a'] + alpha/N * (-log(1 - a'^2 + 1e-6))
    const float du = da[(size_t)row * A + k] * one_m + alpha_invN * 2.f * an * one_m / (one_m + 1e-6f);
    const float dls = du * sig * e - alpha_invN;
    dout[(size_t)row * 2 * A + k] = du;
    dout[(size_t)row * 2 * A + A + k] = (lsr >= kLogSigMin && lsr <= kLogSigMax) ? dls : 0.f;
  }
}

}  // namespace crl

static crl_status mlp_fwd(crl_ctx* ctx, const EncoderPlan& P, const float* prm, const float* x0, int ld0,
                          const float* x0b, int ld0b, int fsplit, float** X, float** Z, float* out, int act,
                          cudaStream_t st, int* nl) {
  const int Bl = ctx->cfg.batch_local;
  for (int l = 0; l < P.n_layers; ++l) {
    const LayerPlan& L = P.layer[l];
    const bool last = l == P.n_layers - 1;
    CU(mlp_forward_layer_f32(Bl, L.in, L.out, l == 0 ? x0 : X[l], l == 0 ? ld0 : L.in, l == 0 ? x0b : nullptr,
                             ld0b, l == 0 ? fsplit : 0, prm + L.w_off, prm + L.b_off, last ? out : Z[l],
                             last ? nullptr : X[l + 1], act, st));
    ++*nl;
  }
  return CRL_OK;
}

__global__ void set_scalar_kernel(float* p, float v) { *p = v; }

// the actor step's schedule; alpha is read from ctx->a_alpha (device) so one captured graph
// serves every alpha (the entropy tuning changes it each step)
static crl_status enqueue_actor(crl_ctx* ctx, const float* s, const float* g, const float* eps, float* loss_out,
                                float* actor_grads_out, int apply_adam, cudaStream_t st) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, A = k.act_dim, D = k.repr_dim, W = k.world_size;
  const float invN = 1.0f / (float)ctx->N;
  const float* cp = ctx->mem.params;              // frozen critic (fp32 master copy)
  const float* ap = ctx->mem.actor_params;
  const size_t na = ctx->sizes.n_actor_params;
  int nl = 0;
  crl_status rs;
  // actor forward on [s || g]
  rs = mlp_fwd(ctx, ctx->actor_plan, ap, s, k.obs_dim, g, k.goal_dim, k.obs_dim, ctx->aX, ctx->aZ, ctx->a_out,
               k.activation, st, &nl);
  if (rs != CRL_OK) return rs;
  const int rb = (Bl + 127) / 128;
  CU(launch_pdl(actor_head_fwd_kernel, dim3(rb), dim3(128), 0, st, Bl, A, (const float*)ctx->a_out, eps,
                ctx->a_new, ctx->a_logpi));
  ++nl;
  // frozen critic on (s, a') and g
  rs = mlp_fwd(ctx, ctx->phi_plan, cp, s, k.obs_dim, ctx->a_new, A, k.obs_dim, ctx->ac_phiX, ctx->ac_phiZ,
               ctx->ac_phi, k.activation, st, &nl);
  if (rs != CRL_OK) return rs;
  rs = mlp_fwd(ctx, ctx->psi_plan, cp, g, k.goal_dim, nullptr, 0, 0, ctx->ac_psiX, ctx->ac_psiZ, ctx->ac_psi,
               k.activation, st, &nl);
  if (rs != CRL_OK) return rs;
  CU(launch_pdl(actor_diag_kernel, dim3((Bl * 32 + 255) / 256), dim3(256), 0, st, Bl, D, k.energy, invN,
                (const float*)ctx->a_alpha, (const float*)ctx->ac_phi, (const float*)ctx->ac_psi, (const float*)ctx->a_logpi,
                ctx->ac_dphi, ctx->a_rowloss));
  ++nl;
  CU(launch_pdl(actor_loss_sum_kernel, dim3(1), dim3(1024), 0, st, Bl, (const float*)ctx->a_rowloss,
                (const float*)ctx->a_logpi, ctx->a_loss));
  ++nl;
  if (ctx->dist) NC(ncclAllReduce(ctx->a_loss, ctx->a_loss, 2, ncclFloat32, ncclSum, ctx->comm, st));
  CU(launch_pdl(actor_loss_finalize_kernel, dim3(1), dim3(1), 0, st, ctx->a_loss, invN, loss_out, ctx->a_skip,
                ctx->a_t, apply_adam, ctx->status));
  ++nl;
  // phi dX chain (critic frozen: no dW), down to the action columns of the input
  {
    const EncoderPlan& P = ctx->phi_plan;
    const float* dZ = ctx->ac_dphi;
    int pp = 0;
    for (int l = P.n_layers - 1; l >= 1; --l) {
      const LayerPlan& L = P.layer[l];
      CU(mlp_backward_dx_f32(Bl, L.in, L.out, dZ, cp + L.w_off, ctx->ac_phiZ[l - 1], ctx->ac_dz[pp], k.activation,
                             st));
      ++nl;
      dZ = ctx->ac_dz[pp];
      pp ^= 1;
    }
    const LayerPlan& L0 = P.layer[0];
    CU(mlp_backward_dx_f32(Bl, A, L0.out, dZ, cp + L0.w_off + (size_t)k.obs_dim * L0.out, nullptr, ctx->a_da,
                           k.activation, st));
    ++nl;
  }
  CU(launch_pdl(actor_head_bwd_kernel, dim3(rb), dim3(128), 0, st, Bl, A, (const float*)ctx->a_alpha, invN,
                (const float*)ctx->a_out, eps, (const float*)ctx->a_new, (const float*)ctx->a_da, ctx->a_dout));
  ++nl;
  // actor backward: dW, db (split-K partials), dX with act'
  {
    const EncoderPlan& P = ctx->actor_plan;
    const float* dZ = ctx->a_dout;
    int pp = 0;
    for (int l = P.n_layers - 1; l >= 0; --l) {
      const LayerPlan& L = P.layer[l];
      CU(mlp_backward_dw_f32(Bl, L.in, L.out, l == 0 ? s : ctx->aX[l], l == 0 ? k.obs_dim : L.in,
                             l == 0 ? g : nullptr, k.goal_dim, l == 0 ? k.obs_dim : 0, dZ, ctx->a_grads + L.w_off,
                             ctx->a_grads + L.b_off, ctx->dw_splits, na, st));
      ++nl;
      if (l > 0) {
        CU(mlp_backward_dx_f32(Bl, L.in, L.out, dZ, ap + L.w_off, ctx->aZ[l - 1], ctx->a_dz[pp], k.activation, st));
        ++nl;
        dZ = ctx->a_dz[pp];
        pp ^= 1;
      }
    }
  }
  if (ctx->dw_splits > 1) {
    CU(launch_reduce_partials(ctx->a_grads, na, ctx->dw_splits, st));
    ++nl;
  }
  if (ctx->dist) NC(ncclAllReduce(ctx->a_grads, ctx->a_grads, na, ncclFloat32, ncclSum, ctx->comm, st));
  if (actor_grads_out)
    CU(cudaMemcpyAsync(actor_grads_out, ctx->a_grads, na * 4, cudaMemcpyDeviceToDevice, st));
  if (apply_adam) {
    CU(launch_adam(ctx->mem.actor_params, ctx->a_grads, 1, ctx->mem.actor_adam_m, ctx->mem.actor_adam_v, na,
                   k.lr_actor, k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay, ctx->a_t, ctx->a_skip, ctx->status,
                   nullptr, ctx->num_sms, st));
    ++nl;
  }
  ctx->launches = nl;
  return CRL_OK;
}

extern "C" crl_status crl_actor_loss(crl_ctx* ctx, const float* s, const float* g, const float* eps,
                                     float alpha_ent, float* loss_out, float* actor_grads_out,
                                     int apply_adam, void* stream) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (!ctx->has_actor) return fail(ctx, CRL_EUNSUPPORTED, "context created without an actor (actor_depth = 0)");
  if (!s || !g || !eps) return fail(ctx, CRL_EINVAL, "actor_loss: NULL s, g or eps");
  if (!(alpha_ent >= 0.f) || !std::isfinite(alpha_ent)) return fail(ctx, CRL_EINVAL, "alpha_ent must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  set_scalar_kernel<<<1, 1, 0, st>>>(ctx->a_alpha, alpha_ent);      // stream-ordered, outside the graph
  CU(cudaGetLastError());
  if (ctx->prof_on || std::getenv("CRL_ACTOR_EAGER")) {
    crl_status rs = enqueue_actor(ctx, s, g, eps, loss_out, actor_grads_out, apply_adam, st);
    if (rs == CRL_OK) ctx->actor_loss_done = true;
    return rs;
  }
  // captured once per (pointers, apply_adam) and replayed: ~20 dependent launches become one
  ActorKey key{s, g, eps, loss_out, actor_grads_out, apply_adam};
  auto it = ctx->actor_graphs.find(key);
  if (it == ctx->actor_graphs.end() && ctx->actor_graphs.size() >= crl_ctx::kMaxGraphs) {
    // bounded cache (as crl_critic_step): evict the least recently replayed actor graph
    auto lru = ctx->actor_graphs.begin();
    for (auto u = ctx->actor_graphs.begin(); u != ctx->actor_graphs.end(); ++u)
      if (ctx->actor_use[u->first] < ctx->actor_use[lru->first]) lru = u;
    cudaGraphExecDestroy(lru->second.first);
    ctx->actor_use.erase(lru->first);
    ctx->actor_graphs.erase(lru);
  }
  if (it == ctx->actor_graphs.end()) {
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    crl_status rs = enqueue_actor(ctx, s, g, eps, loss_out, actor_grads_out, apply_adam, ctx->cap_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (rs != CRL_OK) { if (graph) cudaGraphDestroy(graph); return rs; }
    CU(ce);
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CU(ce);
    it = ctx->actor_graphs.emplace(key, std::make_pair(exec, ctx->launches)).first;
  }
  CU(cudaGraphLaunch(it->second.first, st));
  ctx->actor_use[key] = ++ctx->use_clock;
  ctx->launches = it->second.second;
  ctx->actor_loss_done = true;
  return CRL_OK;
}

// ---------------------------------------------------------------------------------------
// Entropy coefficient ("a tuneable entropy coefficient"; reading A-32): SAC-style
// automatic tuning of alpha = exp(log_alpha) towards a target entropy H,
//   L_alpha = alpha (-E[log pi] - H),   dL_alpha / d log_alpha = alpha (-E[log pi] - H)
// (E[log pi] held constant: it is the mean of the last crl_actor_loss), one Adam step on
// log_alpha with the context's b1 / b2 / eps and no weight decay.
// ---------------------------------------------------------------------------------------
__global__ void entropy_update_kernel(const float* __restrict__ acc, float target, float lr, float b1, float b2,
                                      float eps, float* __restrict__ log_alpha, float* __restrict__ mv,
                                      int* __restrict__ t, float* __restrict__ alpha_out,
                                      float* __restrict__ loss_out, int* __restrict__ status) {
  const float mean_logpi = acc[3];
  const float la = *log_alpha;
  const float alpha = expf(la);
  const float gl = alpha * (-mean_logpi - target);
  if (loss_out) loss_out[0] = gl;
  if (!isfinite(gl)) {
    set_status(status, CRL_ENONFINITE);
    if (alpha_out) alpha_out[0] = alpha;
    return;
  }
  const int tn = *t + 1;
  const float m = b1 * mv[0] + (1.f - b1) * gl;
  const float v = b2 * mv[1] + (1.f - b2) * gl * gl;
  const float mhat = m / (1.f - powf(b1, (float)tn));
  const float vhat = v / (1.f - powf(b2, (float)tn));
  const float la_new = la - lr * (mhat / (sqrtf(vhat) + eps));
  mv[0] = m;
  mv[1] = v;
  *t = tn;
  *log_alpha = la_new;
  if (alpha_out) alpha_out[0] = expf(la_new);
}

extern "C" crl_status crl_entropy_update(crl_ctx* ctx, float target_entropy, float lr, float* log_alpha,
                                         float* alpha_out, float* loss_out, void* stream) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (!ctx->has_actor) return fail(ctx, CRL_EUNSUPPORTED, "context created without an actor (actor_depth = 0)");
  if (!log_alpha) return fail(ctx, CRL_EINVAL, "entropy_update: NULL log_alpha");
  if (!(lr > 0.f) || !std::isfinite(lr) || !std::isfinite(target_entropy))
    return fail(ctx, CRL_EINVAL, "entropy_update: lr must be > 0 and the target finite");
  if (!ctx->actor_loss_done) return fail(ctx, CRL_ESTATE, "entropy_update needs a prior crl_actor_loss");
  const crl_config& k = ctx->cfg;
  cudaStream_t st = (cudaStream_t)stream;
  entropy_update_kernel<<<1, 1, 0, st>>>(ctx->a_loss, target_entropy, lr, k.adam_b1, k.adam_b2, k.adam_eps,
                                         log_alpha, ctx->ent_mv, ctx->ent_t, alpha_out, loss_out, ctx->status);
  CU(cudaGetLastError());
  ctx->launches = 1;
  return CRL_OK;
}
