// crl_api.cu — the C ABI (include/crl.h): context, workspace carving, argument checks, the
// critic-step schedule (captured once per pointer tuple into a CUDA graph and replayed),
// data-parallel collectives over NCCL, device status word.
//
// Critic step schedule (one rank; W = world size, B_l local rows, N = W B_l):
//   phi fwd (d+1 GEMMs, fused bias+act)        psi fwd
//   [W>1] all-gather Phi, Psi (global negatives, reading A-21)
//   LSE_i  = lse_rows(Phi_l, Psi_g)              LSE'_j = lse_rows(Psi_l, Phi_g)
//   [W>1] all-gather LSE, LSE'
//   loss partial sums (+ finalize when W = 1)  [W>1] all-reduce 3 floats + finalize
//   dPhi_l = grad_rows(Phi_l, Psi_g, LSE_l, LSE'_g)   dPsi_l = grad_rows(Psi_l, Phi_g, LSE'_l, LSE_g)
//   phi bwd, psi bwd (dW, db, dX with fused act')
//   [W>1] all-reduce grads (sum; per-row terms already carry 1/N, reading A-23)
//   Adam (+ bf16 shadow)
#include "common.cuh"

#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "ctx.h"

thread_local std::string g_last_error;

crl_status bf16_prepare(crl_ctx* ctx);
crl_status enqueue_critic_bf16(crl_ctx* ctx, const float* s, const float* a, const float* g, float* loss_out,
                               float* grads_out, cudaStream_t st, cudaStream_t st2);

cudaEvent_t pool_event(crl_ctx* c) {
  if (c->ev_pool_next == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_pool_next++];
}

// Profiling only: holds the stream for `ns` so the launches queued behind it run back to
// back on the GPU (the event-bracketed stage times then exclude host enqueue gaps).
__global__ void spin_kernel(unsigned long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}


static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// SM count of the current device (split counts of the logits kernels, hence scratch sizes);
// 148 (B200) when no device is visible (crl_workspace_size is a pure host call)
static int device_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      n <= 0) {
    cudaGetLastError();
    return 148;
  }
  return n;
}

static void carve(crl_ctx* c, char* buf_base, char* scr_base, size_t* buf_bytes,
                  size_t* scr_bytes) {
  const crl_config& k = c->cfg;
  const int E = k.n_envs_local, T = k.capacity;
  c->obs_stride = round_up(k.obs_dim, 4);
  c->act_stride = round_up(k.act_dim, 4);
  Carver b{buf_base};
  c->obs_ring = b.take<float>((size_t)E * T * c->obs_stride);
  c->act_ring = b.take<float>((size_t)E * T * c->act_stride);
  c->ep_end = b.take<uint32_t>((size_t)E * T);
  c->open_start = b.take<uint32_t>((size_t)E);
  c->qtab = b.take<uint64_t>((size_t)T + 1);
  *buf_bytes = (b.off + 255) & ~(size_t)255;

  const int Bl = k.batch_local, W = k.world_size, N = Bl * W, D = k.repr_dim, Wd = k.width;
  const bool dist = W > 1 || force_dist();
  c->dist = dist;
  Carver s{scr_base};
  c->dw_splits = dw_splits_for(Bl);
  // wide encoders (configs[4]: 4 x 1024) already have ~200 weight-gradient tiles per K slice:
  // more slices only add partial-buffer traffic (Adam sums them).  Measured on B200 at
  // netscale: 8 slices 584 steps/s (dW 278 us + Adam 74 us), 2 slices 601 (257 + 48).
  // (A CTA-pair variant of the grouped kernel, 256 x 256 tiles, measured slower at netscale:
  // 668 vs 679 steps/s -- its bias sums double the MMA work of every M-block-0 tile and its
  // single accumulator serialises the epilogue; not kept.)
  if (k.width >= 512 && !std::getenv("CRL_DW_SPLITS")) c->dw_splits = std::min(c->dw_splits, 2);
  c->grads = s.take<float>(c->sizes.n_params * c->dw_splits);
  const bool bf = k.precision == CRL_BF16;
  c->bf16 = bf;
  if (!bf) {
    for (int l = 1; l <= k.depth; ++l) {
      c->phiX[l] = s.take<float>((size_t)Bl * Wd);
      c->psiX[l] = s.take<float>((size_t)Bl * Wd);
    }
    for (int l = 0; l < k.depth; ++l) {
      c->phiZ[l] = s.take<float>((size_t)Bl * Wd);
      if (k.layernorm) {
        c->phiY[l] = s.take<float>((size_t)Bl * Wd); c->psiY[l] = s.take<float>((size_t)Bl * Wd);
        c->phiMu[l] = s.take<float>((size_t)Bl); c->psiMu[l] = s.take<float>((size_t)Bl);
        c->phiRs[l] = s.take<float>((size_t)Bl); c->psiRs[l] = s.take<float>((size_t)Bl);
      }
      c->psiZ[l] = s.take<float>((size_t)Bl * Wd);
    }
  } else {
    // bf16 operands; every row pitch is a multiple of 8 elements (16 B, TMA requirement)
    c->wshadow = s.take<__nv_bfloat16>(c->sizes.n_params);
    c->ld0_phi = round_up(k.obs_dim + k.act_dim, 8);
    c->ld0_psi = round_up(k.goal_dim, 8);
    c->x0_phi = s.take<__nv_bfloat16>((size_t)Bl * c->ld0_phi);
    c->x0_psi = s.take<__nv_bfloat16>((size_t)Bl * c->ld0_psi);
    for (int l = 1; l <= k.depth; ++l) {
      c->phiXb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
      c->psiXb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
    }
    for (int l = 0; l < k.depth; ++l) {
      c->phiZb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
      c->psiZb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
      if (k.layernorm) {                         // F2 on the bf16 path: Y = LN(Z) and its statistics
        c->phiYb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd); c->psiYb[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
        c->phiMu[l] = s.take<float>((size_t)Bl); c->psiMu[l] = s.take<float>((size_t)Bl);
        c->phiRs[l] = s.take<float>((size_t)Bl); c->psiRs[l] = s.take<float>((size_t)Bl);
      }
    }
    if (k.layernorm) {                           // per-CTA dgamma / dbeta partials, one set per encoder
      c->ln_nblk = 2 * device_sms();
      c->ln_part_phi = s.take<float>((size_t)c->ln_nblk * 2 * Wd);
      c->ln_part_psi = s.take<float>((size_t)c->ln_nblk * 2 * Wd);
    }
    c->phi_outb = s.take<__nv_bfloat16>((size_t)Bl * D);
    c->psi_outb = s.take<__nv_bfloat16>((size_t)Bl * D);
    c->dphib = s.take<__nv_bfloat16>((size_t)Bl * D);
    c->dpsib = s.take<__nv_bfloat16>((size_t)Bl * D);
    for (int l = 0; l < k.depth; ++l) {          // dZ_l of hidden layer l: [B][width]
      c->dzb_phi[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
      c->dzb_psi[l] = s.take<__nv_bfloat16>((size_t)Bl * Wd);
    }
    // CRL_TC_LOGITS_MIN_N overrides the SIMT/tensor-core crossover (measurement knob)
    const char* mn = std::getenv("CRL_TC_LOGITS_MIN_N");
    c->tc_logits = N >= (mn ? std::atoi(mn) : kTcLogitsMinN) && tc_logits_supports(D);
    if (c->tc_logits) {
      // both sides share the SMs (one two-sided statistics launch; the two gradient calls run
      // concurrently): the split count minimises the makespan on half of them each
      c->lg_splits = tc_logits_splits(Bl, N, D, device_sms() / 2);
      if (dist) {
        c->phi_outb_g = s.take<__nv_bfloat16>((size_t)N * D);
        c->psi_outb_g = s.take<__nv_bfloat16>((size_t)N * D);
      } else {
        c->phi_outb_g = c->phi_outb;
        c->psi_outb_g = c->psi_outb;
      }
      c->stat_phi = s.take<float>((size_t)N + kStatPad);
      c->stat_psi = s.take<float>((size_t)N + kStatPad);
      c->fac_ok = s.take<int>(4);
      c->fac_row = s.take<float>((size_t)Bl + kStatPad);
      c->fac_col = s.take<float>((size_t)Bl + kStatPad);
      if (dist) {
        c->fac_row_g = s.take<float>((size_t)N + kStatPad);
        c->fac_col_g = s.take<float>((size_t)N + kStatPad);
      } else {
        c->fac_row_g = c->fac_row;
        c->fac_col_g = c->fac_col;
      }
      // two sets (row call on phi, column call on psi run concurrently)
      c->lg_part_m = s.take<float>((size_t)2 * c->lg_splits * Bl);
      c->lg_part_s = s.take<float>((size_t)2 * c->lg_splits * Bl);
      c->lg_part_rs = s.take<float>((size_t)2 * c->lg_splits * Bl);
      c->lg_part_da = s.take<float>((size_t)2 * c->lg_splits * Bl * D);
      c->lg_ticket = s.take<int>((size_t)2 * ((Bl + 127) / 128));
      // one-pass statistics also at W > 1: each rank's column partials are all-reduced (C2)
      c->use_stats = tc_stats_supports(D, k.energy) && !std::getenv("CRL_NO_FUSED_STATS");
      if (c->use_stats) {
        c->st_splits = tc_stats_splits(Bl, N, device_sms());
        c->st_ldc = N + kStatPad;
        c->st_part_rs = s.take<float>((size_t)c->st_splits * Bl);
        c->st_colpart = s.take<float>((size_t)((Bl + 127) / 128) * c->st_ldc);
        c->st_bad = s.take<int>(4);
        if (dist) c->st_colsum = s.take<float>((size_t)N + kStatPad);
      }
      c->use_gradf = !dist && tc_gradf_supports(D, k.energy) && !std::getenv("CRL_NO_FUSED_GRAD");
      if (c->use_gradf) {
        c->gf_splits = tc_gradf_splits(Bl, N, device_sms());
        c->gf_part_da = s.take<float>((size_t)c->gf_splits * Bl * D);
        c->gf_part_rs = s.take<float>((size_t)c->gf_splits * Bl);
        c->gf_acc_bytes = ((size_t)N * D + N + kStatPad) * 4;
        c->gf_acc = s.take<float>(c->gf_acc_bytes / 4);
        c->gf_cs = c->gf_acc + (size_t)N * D;
      }
      // D = 256 (configs[4]): both gradient sides in one persistent launch (tc_grad2.cu)
      c->use_grad2 = D == 256 && !c->use_gradf && !std::getenv("CRL_NO_GRAD2");
      if (c->use_grad2) {
        // CTA pairs (tc_grad2p) once a pair has two full row blocks to share the B tile over
        c->g2_pair = Bl >= 256 && !std::getenv("CRL_NO_GRAD2P");
        c->g2_grid = c->g2_pair ? tc::tc_grad2p_grid(Bl, device_sms()) : tc::tc_grad2_grid(Bl, device_sms());
        // W = 1 and a symmetric energy: side 1 as W^T Phi from the stored W (CRL_NO_G2_WSYM: off)
        c->g2_wsym = c->g2_pair && !dist && N == Bl && k.energy != CRL_ENERGY_COS && tc::pdw_supported(Bl, 2) &&
                     !std::getenv("CRL_NO_G2_WSYM");
        // partial slots: both sides x 2, or (stored W) side 0 x 3 (a pair covers >= half a row-block
        // pair, so a row block is cut into at most 3 pieces) + the 2 K slices of W^T Phi
        c->g2_part_da = s.take<float>((size_t)(c->g2_wsym ? 5 : 4) * Bl * D);
        c->g2_part_rs = s.take<float>((size_t)16 * Bl);   // 2 sides x 2 slots (or 3 slots) x <= 4 sub-slots
        c->g2_flags = s.take<unsigned char>((size_t)2 * ((Bl + 127) / 128));
        if (c->g2_wsym) {
          c->g2_W = s.take<__nv_bfloat16>((size_t)Bl * ((N + 63) / 64 * 64));   // rows padded to 128 B
          c->g2_cs = s.take<float>((size_t)2 * N);
        }
      }
    }
  }
  c->phi_out = s.take<float>((size_t)Bl * D);
  c->psi_out = s.take<float>((size_t)Bl * D);
  if (dist) {
    c->phi_g = s.take<float>((size_t)N * D);
    c->psi_g = s.take<float>((size_t)N * D);
  } else {
    c->phi_g = c->phi_out;
    c->psi_g = c->psi_out;
  }
  // padded: the tensor-core logits read column statistics with 1-D bulk copies of whole tiles
  c->lse_row = s.take<float>((size_t)Bl + kStatPad);
  c->lse_col = s.take<float>((size_t)Bl + kStatPad);
  if (dist) {
    c->lse_row_g = s.take<float>((size_t)N + kStatPad);
    c->lse_col_g = s.take<float>((size_t)N + kStatPad);
  } else {
    c->lse_row_g = c->lse_row;
    c->lse_col_g = c->lse_col;
  }
  c->dphi = s.take<float>((size_t)Bl * D);
  c->dpsi = s.take<float>((size_t)Bl * D);
  const int wmax = Wd > D ? Wd : D;
  if (!bf) {
    c->dz[0] = s.take<float>((size_t)Bl * wmax);
    c->dz[1] = s.take<float>((size_t)Bl * wmax);
    c->dz_psi[0] = s.take<float>((size_t)Bl * wmax);
    c->dz_psi[1] = s.take<float>((size_t)Bl * wmax);
  }
  c->loss_acc = s.take<float>(16);
  if (k.loss >= CRL_LOSS_FB) {
    c->pair_d = s.take<float>((size_t)Bl + kStatPad);
    c->pair_R = s.take<float>((size_t)Bl + kStatPad);
    c->pair_L = s.take<float>((size_t)Bl + kStatPad);
  }
  // loss partials: the loss kernel's CTAs (16 rows each) or the merge's row-side CTAs (8 rows)
  c->loss_part = s.take<float>((size_t)4 * std::max(loss_partial_blocks(Bl), (Bl + 7) / 8));
  c->loss_ticket = s.take<unsigned>(1);
  c->loss_dev = s.take<float>(4);
  c->status = s.take<int>(1);
  c->adam_t = s.take<int>(1);
  c->skip = s.take<int>(1);
  c->stage_s = s.take<float>((size_t)Bl * k.obs_dim);
  c->stage_a = s.take<float>((size_t)Bl * k.act_dim);
  c->stage_g = s.take<float>((size_t)Bl * k.goal_dim + 64);   // + 256 B: the host ring's slot pitch
  // the second staging set: the same three takes, so the same layout (offsets of a and g from s;
  // pointer differences would be 0 in the sizing pass, where the carver has no base)
  c->stage2 = s.take<float>((size_t)Bl * k.obs_dim);
  s.take<float>((size_t)Bl * k.act_dim);
  s.take<float>((size_t)Bl * k.goal_dim + 64);
  // actor objective (fp32): actor activations, the frozen critic's activations on [s||a'],
  // head buffers, gradient partials
  c->has_actor = k.actor_depth > 0 && k.actor_width > 0;
  if (c->has_actor) {
    const int A = k.act_dim, Wa = k.actor_width;
    c->actor_plan = make_encoder_plan(k.obs_dim + k.goal_dim, k.actor_depth, Wa, 2 * A, 0);
    for (int l = 1; l <= k.actor_depth; ++l) c->aX[l] = s.take<float>((size_t)Bl * Wa);
    for (int l = 0; l < k.actor_depth; ++l) c->aZ[l] = s.take<float>((size_t)Bl * Wa);
    c->a_out = s.take<float>((size_t)Bl * 2 * A);
    c->a_new = s.take<float>((size_t)Bl * A);
    c->a_logpi = s.take<float>((size_t)Bl);
    c->a_rowloss = s.take<float>((size_t)Bl);
    c->a_dout = s.take<float>((size_t)Bl * 2 * A);
    c->a_da = s.take<float>((size_t)Bl * A);
    const int wa = Wa > 2 * A ? Wa : 2 * A;
    c->a_dz[0] = s.take<float>((size_t)Bl * wa);
    c->a_dz[1] = s.take<float>((size_t)Bl * wa);
    for (int l = 1; l <= k.depth; ++l) {
      c->ac_phiX[l] = s.take<float>((size_t)Bl * Wd);
      c->ac_psiX[l] = s.take<float>((size_t)Bl * Wd);
    }
    for (int l = 0; l < k.depth; ++l) {
      c->ac_phiZ[l] = s.take<float>((size_t)Bl * Wd);
      c->ac_psiZ[l] = s.take<float>((size_t)Bl * Wd);
    }
    c->ac_phi = s.take<float>((size_t)Bl * D);
    c->ac_psi = s.take<float>((size_t)Bl * D);
    c->ac_dphi = s.take<float>((size_t)Bl * D);
    c->ac_dz[0] = s.take<float>((size_t)Bl * wmax);
    c->ac_dz[1] = s.take<float>((size_t)Bl * wmax);
    c->a_grads = s.take<float>(c->actor_plan.n_params * c->dw_splits);
    c->a_loss = s.take<float>(4);
    c->a_t = s.take<int>(1);
    c->a_skip = s.take<int>(1);
    c->a_alpha = s.take<float>(1);
    c->ent_mv = s.take<float>(2);
    c->ent_t = s.take<int>(1);
  }
  *scr_bytes = (s.off + 255) & ~(size_t)255;
}

static bool make_host_ring(crl_ctx* ctx);

// device-side pull of a page-locked host slot (UVA), 16 B per load
__global__ void pull_host_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

static crl_status validate(const crl_config* k, crl_ctx* ctx) {
  if (!k) return fail(ctx, CRL_EINVAL, "cfg is NULL");
  if (k->obs_dim <= 0 || k->act_dim <= 0 || k->goal_dim <= 0)
    return fail(ctx, CRL_EINVAL, "obs_dim, act_dim and goal_dim must be positive");
  if (k->goal_offset < 0 || k->goal_offset + k->goal_dim > k->obs_dim)
    return fail(ctx, CRL_EINVAL, "goal slice obs[goal_offset:goal_offset+goal_dim] out of range");
  if (k->n_envs_local <= 0 || k->capacity < 2)
    return fail(ctx, CRL_EINVAL, "n_envs_local must be > 0 and capacity >= 2");
  if (!(k->gamma >= 0.0 && k->gamma < 1.0)) return fail(ctx, CRL_EINVAL, "gamma must be in [0, 1)");
  if (k->depth < 0 || k->depth > CRL_MAX_LAYERS - 1 || k->width <= 0)
    return fail(ctx, CRL_EINVAL, "depth must be in [0, 7] and width > 0");
  if (!logits_simt_supports(k->repr_dim))
    return fail(ctx, CRL_EUNSUPPORTED, "repr_dim must be one of 16, 32, 64, 128, 256");
  if (k->activation != CRL_ACT_SILU && k->activation != CRL_ACT_RELU)
    return fail(ctx, CRL_EINVAL, "activation");
  if (k->energy < 0 || k->energy > 4) return fail(ctx, CRL_EINVAL, "energy");
  if (k->precision == CRL_BF16 && k->energy == CRL_ENERGY_L1)
    return fail(ctx, CRL_EUNSUPPORTED, "the L1 energy (not a contraction) runs on the fp32 path only");
  if (k->loss < 0 || k->loss > 8) return fail(ctx, CRL_EINVAL, "loss");
  if (k->loss >= CRL_LOSS_FB && (k->precision != CRL_FP32 || k->world_size != 1))
    return fail(ctx, CRL_EUNSUPPORTED, "FB / DPO / IPO / SPPO run on the fp32 path with world_size 1");
  if (k->precision != CRL_FP32 && k->precision != CRL_BF16) return fail(ctx, CRL_EINVAL, "precision");
  if (k->layernorm != 0 && k->layernorm != 1) return fail(ctx, CRL_EINVAL, "layernorm must be 0 or 1");
  if (!(k->random_goal_alpha >= 0.f && k->random_goal_alpha <= 1.f))
    return fail(ctx, CRL_EINVAL, "random_goal_alpha must be in [0, 1]");
  if (k->layernorm && k->precision == CRL_FP32 && k->width > 2048)
    return fail(ctx, CRL_EUNSUPPORTED, "LayerNorm encoders on the fp32 path need width <= 2048");
  if (k->layernorm && k->precision == CRL_BF16 &&
      !(ln_bf16_supports(k->width) && (long long)k->batch_local >= 256))
    return fail(ctx, CRL_EUNSUPPORTED, "LayerNorm encoders on the bf16 path need width in {256, 512, 768, 1024} "
                                       "and batch_local >= 256 (CTA-pair GEMMs for every hidden layer)");
  if (k->layernorm && k->actor_depth > 0)
    return fail(ctx, CRL_EUNSUPPORTED, "the actor's frozen-critic pass has no LayerNorm encoders");
  if (k->precision == CRL_BF16 && (k->width % 16 != 0))
    return fail(ctx, CRL_EUNSUPPORTED, "bf16 path needs width % 16 == 0");
  if (k->world_size < 1 || k->rank < 0 || k->rank >= k->world_size)
    return fail(ctx, CRL_EINVAL, "rank / world_size");
  if (k->batch_local < 1 || (long long)k->batch_local * k->world_size < 2)
    return fail(ctx, CRL_EINVAL, "global batch must be >= 2 (InfoNCE needs negatives)");
  if (!(k->lr > 0.f) || !(k->adam_eps > 0.f)) return fail(ctx, CRL_EINVAL, "lr and eps must be > 0");
  if (k->actor_depth < 0 || k->actor_depth > CRL_MAX_LAYERS - 1 || k->actor_width < 0)
    return fail(ctx, CRL_EINVAL, "actor_depth must be in [0, 7] and actor_width >= 0");
  if (k->actor_depth > 0 && k->actor_width > 0 && !(k->lr_actor > 0.f))
    return fail(ctx, CRL_EINVAL, "lr_actor must be > 0");
  return CRL_OK;
}

extern "C" {

int crl_abi_version(void) { return CRL_ABI_VERSION; }

const char* crl_last_error(const crl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

crl_status crl_workspace_size(const crl_config* cfg, crl_sizes* out) {
  crl_ctx* ctx = nullptr;
  crl_status st = validate(cfg, ctx);
  if (st != CRL_OK) return st;
  if (!out) return fail(ctx, CRL_EINVAL, "out is NULL");
  crl_ctx tmp;
  tmp.cfg = *cfg;
  tmp.phi_plan = make_encoder_plan(cfg->obs_dim + cfg->act_dim, cfg->depth, cfg->width,
                                   cfg->repr_dim, 0, cfg->layernorm != 0);
  tmp.psi_plan = make_encoder_plan(cfg->goal_dim, cfg->depth, cfg->width, cfg->repr_dim,
                                   tmp.phi_plan.n_params, cfg->layernorm != 0);
  tmp.sizes.n_params = tmp.phi_plan.n_params + tmp.psi_plan.n_params;
  if (cfg->actor_depth > 0 && cfg->actor_width > 0) {
    EncoderPlan a = make_encoder_plan(cfg->obs_dim + cfg->goal_dim, cfg->actor_depth,
                                      cfg->actor_width, 2 * cfg->act_dim, 0);
    tmp.sizes.n_actor_params = a.n_params;
  }
  carve(&tmp, nullptr, nullptr, &tmp.sizes.buffer_bytes, &tmp.sizes.scratch_bytes);
  *out = tmp.sizes;
  return CRL_OK;
}

crl_status crl_nccl_unique_id(void* out128) {
  crl_ctx* ctx = nullptr;
  if (!out128) return fail(ctx, CRL_EINVAL, "out128 is NULL");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return CRL_OK;
}

crl_status crl_create(const crl_config* cfg, const crl_memory* mem, const void* nccl_id,
                      crl_ctx** out) {
  crl_ctx* ctx = nullptr;
  crl_status st = validate(cfg, ctx);
  if (st != CRL_OK) return st;
  if (!mem || !out || !mem->params || !mem->adam_m || !mem->adam_v || !mem->buffer || !mem->scratch)
    return fail(ctx, CRL_EINVAL, "memory pointers must be non-NULL");
  if (((uintptr_t)mem->buffer & 255) || ((uintptr_t)mem->scratch & 255))
    return fail(ctx, CRL_EINVAL, "buffer and scratch must be 256-byte aligned");
  if (cfg->world_size > 1 && !nccl_id)
    return fail(ctx, CRL_EINVAL, "world_size > 1 needs an NCCL unique id");
  if (cfg->actor_depth > 0 && cfg->actor_width > 0 &&
      (!mem->actor_params || !mem->actor_adam_m || !mem->actor_adam_v))
    return fail(ctx, CRL_EINVAL, "actor configured: actor_params / actor_adam_m / actor_adam_v must be non-NULL");
  crl_sizes sz;
  st = crl_workspace_size(cfg, &sz);
  if (st != CRL_OK) return st;

  ctx = new crl_ctx();
  ctx->cfg = *cfg;
  ctx->sizes = sz;
  ctx->mem = *mem;
  ctx->N = cfg->batch_local * cfg->world_size;
  ctx->phi_plan = make_encoder_plan(cfg->obs_dim + cfg->act_dim, cfg->depth, cfg->width,
                                    cfg->repr_dim, 0, cfg->layernorm != 0);
  ctx->psi_plan = make_encoder_plan(cfg->goal_dim, cfg->depth, cfg->width, cfg->repr_dim,
                                    ctx->phi_plan.n_params, cfg->layernorm != 0);
  size_t bb, sb;
  carve(ctx, (char*)mem->buffer, (char*)mem->scratch, &bb, &sb);

  auto cleanup = [&](crl_status s) { crl_status r = s; delete ctx; return r; };
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return cleanup(fail(nullptr, CRL_ECUDA, "no CUDA device"));
  gemm_set_num_sms(ctx->num_sms);
  logits_set_num_sms(ctx->num_sms);

  // geometric offset table (contract C1): G[k] = gamma^k by repeated multiplication,
  // Q[k] = floor((1 - G[k]) 2^64), saturated.
  std::vector<uint64_t> q(cfg->capacity + 1);
  double G = 1.0;
  for (int k = 0; k <= cfg->capacity; ++k) {
    if (k > 0) G = G * cfg->gamma;
    double x = 1.0 - G;
    q[k] = (x >= 1.0) ? ~0ull : (uint64_t)(x * 18446744073709551616.0);
  }
  if (cudaMemcpy(ctx->qtab, q.data(), q.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(ctx->ep_end, 0xFF, (size_t)cfg->n_envs_local * cfg->capacity * 4) != cudaSuccess ||
      cudaMemset(ctx->open_start, 0, (size_t)cfg->n_envs_local * 4) != cudaSuccess ||
      cudaMemset(ctx->status, 0, 4) != cudaSuccess || cudaMemset(ctx->adam_t, 0, 4) != cudaSuccess ||
      cudaMemset(ctx->skip, 0, 4) != cudaSuccess || cudaMemset(ctx->loss_ticket, 0, 4) != cudaSuccess ||
      (ctx->lg_ticket && cudaMemset(ctx->lg_ticket, 0, (size_t)2 * ((cfg->batch_local + 127) / 128) * 4) != cudaSuccess) ||
      (ctx->has_actor && (cudaMemset(ctx->a_t, 0, 4) != cudaSuccess || cudaMemset(ctx->a_skip, 0, 4) != cudaSuccess ||
                          cudaMemset(ctx->ent_mv, 0, 8) != cudaSuccess || cudaMemset(ctx->ent_t, 0, 4) != cudaSuccess)) ||
      cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->cap_stream3, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->cap_stream4, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->cap_body, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      !make_host_ring(ctx) ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return cleanup(fail(nullptr, CRL_ECUDA, "context initialisation failed"));
  if (ctx->dist) {
    const char* nb = std::getenv("CRL_AR_BUCKETS");
    ctx->ar_buckets = std::max(1, std::min(crl_ctx::kMaxArBuckets, nb ? std::atoi(nb) : 4));
    ctx->ev_bkt.resize(2 * crl_ctx::kMaxArBuckets, nullptr);
    for (auto& e : ctx->ev_bkt)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        return cleanup(fail(nullptr, CRL_ECUDA, "context initialisation failed (bucket events)"));
  }

  if (ctx->bf16) {
    crl_status bs = bf16_prepare(ctx);
    if (bs != CRL_OK) { std::string m = ctx->err; delete ctx; return fail(nullptr, bs, m); }
  }
  if (ctx->dist) {
    ncclUniqueId id;
    if (cfg->world_size > 1) {
      std::memcpy(&id, nccl_id, sizeof(id));
    } else if (ncclGetUniqueId(&id) != ncclSuccess) {   // CRL_FORCE_DIST: a one-rank communicator
      return cleanup(fail(nullptr, CRL_ENCCL, "ncclGetUniqueId failed"));
    }
    ncclResult_t r = ncclCommInitRank(&ctx->comm, cfg->world_size, id, cfg->rank);
    if (r != ncclSuccess)
      return cleanup(fail(nullptr, CRL_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
  }
  *out = ctx;
  return CRL_OK;
}

crl_status crl_destroy(crl_ctx* ctx) {
  if (!ctx) return CRL_OK;
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : ctx->actor_graphs) cudaGraphExecDestroy(kv.second.first);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->cap_stream2) cudaStreamDestroy(ctx->cap_stream2);
  if (ctx->cap_stream3) cudaStreamDestroy(ctx->cap_stream3);
  if (ctx->cap_stream4) cudaStreamDestroy(ctx->cap_stream4);
  if (ctx->cap_body) cudaStreamDestroy(ctx->cap_body);
  if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
  for (auto e : ctx->ev_bkt)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  for (int i = 0; i < crl_ctx::kHostSlots; ++i)
    if (ctx->h_ev[i]) cudaEventDestroy(ctx->h_ev[i]);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (int d = 0; d < 2; ++d) {
    if (ctx->ev_dcopied[d]) cudaEventDestroy(ctx->ev_dcopied[d]);
    if (ctx->ev_dfree[d]) cudaEventDestroy(ctx->ev_dfree[d]);
  }
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
  return CRL_OK;
}

crl_status crl_get_status(crl_ctx* ctx, int sync, int reset) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (sync) CU(cudaDeviceSynchronize());
  int h = 0;
  CU(cudaMemcpy(&h, ctx->status, 4, cudaMemcpyDeviceToHost));
  if (reset) CU(cudaMemset(ctx->status, 0, 4));
  return (crl_status)h;
}

int crl_last_launch_count(const crl_ctx* ctx) { return ctx ? ctx->launches : 0; }

crl_status crl_debug_tensor(crl_ctx* ctx, const char* name, const float** ptr, size_t* count) {
  if (!ctx || !name || !ptr || !count) return fail(ctx, CRL_EINVAL, "NULL argument");
  const size_t Bl = ctx->cfg.batch_local, D = ctx->cfg.repr_dim;
  std::string n(name);
  if (n == "phi") { *ptr = ctx->phi_out; *count = Bl * D; }
  else if (n == "psi") { *ptr = ctx->psi_out; *count = Bl * D; }
  else if (n == "lse_row") { *ptr = ctx->lse_row; *count = Bl; }
  else if (n == "lse_col") { *ptr = ctx->lse_col; *count = Bl; }
  else if (n == "dphi") { *ptr = ctx->dphi; *count = Bl * D; }
  else if (n == "dpsi") { *ptr = ctx->dpsi; *count = Bl * D; }
  else if (n == "grads") { *ptr = ctx->grads; *count = ctx->sizes.n_params; }
  else if (n == "loss") { *ptr = ctx->loss_dev; *count = 4; }
  else return fail(ctx, CRL_EINVAL, "unknown debug tensor " + n);
  return CRL_OK;
}

crl_status crl_buffer_insert(crl_ctx* ctx, const float* obs, const float* act, const uint8_t* done,
                             int U, void* stream) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (!obs || !act || !done || U <= 0) return fail(ctx, CRL_EINVAL, "insert: NULL input or U <= 0");
  const crl_config& k = ctx->cfg;
  if (ctx->n_ins + (uint64_t)U >= 0xFFFFFFF0ull) return fail(ctx, CRL_ESTATE, "step counter overflow");
  CU(launch_buffer_insert(obs, act, done, U, k.n_envs_local, k.capacity, k.obs_dim, k.act_dim,
                          ctx->obs_stride, ctx->act_stride, (uint32_t)ctx->n_ins, ctx->obs_ring,
                          ctx->act_ring, ctx->ep_end, ctx->open_start, (cudaStream_t)stream));
  ctx->n_ins += (uint64_t)U;
  ctx->launches = 1;
  return CRL_OK;
}

static crl_status relabel(crl_ctx* ctx, uint64_t seed, uint64_t step, int n_upd, float* s, float* a, float* g,
                          float* g_actor, int64_t* idx, void* stream) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (!s || !a || !g) return fail(ctx, CRL_EINVAL, "sample: NULL output");
  if (n_upd < 1 || (long)n_upd * ctx->cfg.batch_local > (1l << 30))
    return fail(ctx, CRL_EINVAL, "sample: n_updates must be >= 1 and n_updates * batch_local <= 2^30");
  const crl_config& k = ctx->cfg;
  const uint64_t n_ins = ctx->n_ins;
  const uint64_t tau_new = n_ins - 1;
  const uint64_t tau_old = n_ins > (uint64_t)k.capacity ? n_ins - k.capacity : 0;
  if (n_ins < 2) return fail(ctx, CRL_ESTATE, "buffer holds fewer than 2 slots per env");
  if (ctx->prof_on) spin_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(100000ull);
  Stage sg(ctx, (cudaStream_t)stream, n_upd > 1 ? "relabel_bulk" : "relabel");
  CU(launch_relabel_sample(k.batch_local, n_upd, k.rank, k.n_envs_local, k.capacity, k.obs_dim, k.act_dim,
                           k.goal_dim, k.goal_offset, ctx->obs_stride, ctx->act_stride,
                           (uint32_t)tau_old, (uint32_t)tau_new, seed, step, k.gamma,
                           (uint64_t)((double)k.random_goal_alpha * 4294967296.0), ctx->obs_ring,
                           ctx->act_ring, ctx->ep_end, ctx->qtab, s, a, g, g_actor, idx, ctx->status,
                           (cudaStream_t)stream));
  ctx->launches = 1;
  return CRL_OK;
}

crl_status crl_relabel_sample(crl_ctx* ctx, uint64_t seed, uint64_t step, float* s, float* a,
                              float* g, int64_t* idx, void* stream) {
  return relabel(ctx, seed, step, 1, s, a, g, nullptr, idx, stream);
}

crl_status crl_relabel_sample_bulk(crl_ctx* ctx, uint64_t seed, uint64_t step0, int n_updates, float* s,
                                   float* a, float* g, int64_t* idx, void* stream) {
  return relabel(ctx, seed, step0, n_updates, s, a, g, nullptr, idx, stream);
}

crl_status crl_relabel_sample_mixed(crl_ctx* ctx, uint64_t seed, uint64_t step0, int n_updates, float* s,
                                    float* a, float* g, float* g_actor, int64_t* idx, void* stream) {
  if (ctx && !g_actor) return fail(ctx, CRL_EINVAL, "sample_mixed: NULL g_actor");
  return relabel(ctx, seed, step0, n_updates, s, a, g, g_actor, idx, stream);
}

}  // extern "C"

// ----------------------------------------------------------------------------------------
// critic step
// ----------------------------------------------------------------------------------------
static crl_status enc_forward(crl_ctx* ctx, const char* tag, const EncoderPlan& P, const float* x0, int ld0,
                              const float* x0b, int ld0b, int fsplit, float** X, float** Z,
                              float* out, cudaStream_t st, int* nl) {
  const crl_config& k = ctx->cfg;
  const float* prm = ctx->mem.params;
  const int Bl = k.batch_local;
  const bool ln = k.layernorm != 0;               // F2: Z -> LayerNorm -> act (ln.cu)
  float** Y = X == ctx->phiX ? ctx->phiY : ctx->psiY;
  float** Mu = X == ctx->phiX ? ctx->phiMu : ctx->psiMu;
  float** Rs = X == ctx->phiX ? ctx->phiRs : ctx->psiRs;
  for (int l = 0; l < P.n_layers; ++l) {
    const LayerPlan& L = P.layer[l];
    const bool last = (l == P.n_layers - 1);
    const float* xin = (l == 0) ? x0 : X[l];
    const int ldx = (l == 0) ? ld0 : L.in;
    Stage sg(ctx, st, std::string(tag) + "_fwd_l" + std::to_string(l));
    CU(mlp_forward_layer_f32(Bl, L.in, L.out, xin, ldx, l == 0 ? x0b : nullptr, ld0b,
                             l == 0 ? fsplit : 0, prm + L.w_off, prm + L.b_off,
                             last ? out : Z[l], (last || ln) ? nullptr : X[l + 1], k.activation, st));
    ++*nl;
    if (ln && !last) {
      CU(launch_ln_fwd(Bl, L.out, Z[l], prm + L.g_off, prm + L.be_off, k.activation, Y[l], X[l + 1], Mu[l], Rs[l],
                       st));
      ++*nl;
    }
  }
  return CRL_OK;
}

static crl_status enc_backward(crl_ctx* ctx, const char* tag, const EncoderPlan& P, const float* x0, int ld0,
                               const float* x0b, int ld0b, int fsplit, float** X, float** Z,
                               const float* dY, float** dzbuf, cudaStream_t st, int* nl) {
  const crl_config& k = ctx->cfg;
  const float* prm = ctx->mem.params;
  const int Bl = k.batch_local;
  const bool ln = k.layernorm != 0;
  float** Yl = X == ctx->phiX ? ctx->phiY : ctx->psiY;
  float** Mu = X == ctx->phiX ? ctx->phiMu : ctx->psiMu;
  float** Rs = X == ctx->phiX ? ctx->phiRs : ctx->psiRs;
  const float* dZ = dY;
  int pp = 0;
  for (int l = P.n_layers - 1; l >= 0; --l) {
    const LayerPlan& L = P.layer[l];
    const float* xin = (l == 0) ? x0 : X[l];
    const int ldx = (l == 0) ? ld0 : L.in;
    {
      Stage sg(ctx, st, std::string(tag) + "_bwd_dw_l" + std::to_string(l));
      CU(mlp_backward_dw_f32(Bl, L.in, L.out, xin, ldx, l == 0 ? x0b : nullptr, ld0b,
                             l == 0 ? fsplit : 0, dZ, ctx->grads + L.w_off, ctx->grads + L.b_off,
                             ctx->dw_splits, ctx->sizes.n_params, st));
    }
    ++*nl;
    if (l > 0) {
      float* dst = dzbuf[pp];
      Stage sg(ctx, st, std::string(tag) + "_bwd_dx_l" + std::to_string(l));
      // dX * act'(.) at the pre-activation: Z_{l-1}, or with LayerNorm Y_{l-1} (then dY -> dZ)
      CU(mlp_backward_dx_f32(Bl, L.in, L.out, dZ, prm + L.w_off, ln ? Yl[l - 1] : Z[l - 1], dst, k.activation, st));
      ++*nl;
      if (ln) {
        const LayerPlan& Lp = P.layer[l - 1];
        CU(launch_ln_bwd(Bl, Lp.out, dst, Z[l - 1], Mu[l - 1], Rs[l - 1], prm + Lp.g_off, ctx->grads + Lp.g_off,
                         ctx->grads + Lp.be_off, ctx->dw_splits, ctx->sizes.n_params, st));
        ++*nl;
      }
      dZ = dst;
      pp ^= 1;
    }
  }
  return CRL_OK;
}

// Fork/join helpers: during graph capture the phi and psi chains run on two streams
// (independent until the logits), which shortens the critical path of a latency-bound step.
static void fork(crl_ctx* ctx, cudaStream_t s0, cudaStream_t s1) {
  if (s0 == s1) return;
  cudaEventRecord(ctx->ev_fork, s0);
  cudaStreamWaitEvent(s1, ctx->ev_fork, 0);
}
static void join(crl_ctx* ctx, cudaStream_t s0, cudaStream_t s1) {
  if (s0 == s1) return;
  cudaEventRecord(ctx->ev_join, s1);
  cudaStreamWaitEvent(s0, ctx->ev_join, 0);
}

crl_status crl::enqueue_allreduce_adam(crl_ctx* ctx, cudaStream_t st, cudaStream_t st2, void* shadow, int keep_sum,
                                  int* nl) {
  const crl_config& k = ctx->cfg;
  const size_t n = ctx->sizes.n_params;
  if (!ctx->dist && ctx->pdw_split) {
    // phi's parameters [0, lo) after phi's dW launch (st), the rest after psi's (st2, which also
    // waits for st: [lo, n_phi) is phi's when n_phi is not a multiple of 256)
    const size_t lo = (size_t)ctx->phi_plan.n_params / 256 * 256;
    cudaEventRecord(ctx->ev_side, st);
    if (st2 != st) cudaStreamWaitEvent(st2, ctx->ev_side, 0);
    {
      Stage sg(ctx, st, "adam");
      CU(launch_adam_range(ctx->mem.params, ctx->grads, ctx->dw_splits, n, ctx->mem.adam_m, ctx->mem.adam_v, lo,
                           k.lr, k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay, ctx->adam_t, ctx->skip,
                           ctx->status, shadow, ctx->num_sms, keep_sum, st));
    }
    CU(launch_adam_range(ctx->mem.params + lo, ctx->grads + lo, ctx->dw_splits, n, ctx->mem.adam_m + lo,
                         ctx->mem.adam_v + lo, n - lo, k.lr, k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay,
                         ctx->adam_t, ctx->skip, ctx->status,
                         shadow ? static_cast<void*>(static_cast<__nv_bfloat16*>(shadow) + lo) : nullptr,
                         ctx->num_sms, keep_sum, st2));
    if (st2 != st) {
      cudaEventRecord(ctx->ev_join, st2);
      cudaStreamWaitEvent(st, ctx->ev_join, 0);
    }
    *nl += 2;
    return CRL_OK;
  }
  if (!ctx->dist) {
    Stage sg(ctx, st, "adam");
    CU(launch_adam_ex(ctx->mem.params, ctx->grads, ctx->dw_splits, ctx->mem.adam_m, ctx->mem.adam_v, n, k.lr,
                      k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay, ctx->adam_t, ctx->skip, ctx->status, shadow,
                      ctx->num_sms, keep_sum, st));
    ++*nl;
    return CRL_OK;
  }
  // buckets of the flat gradient (256-float aligned): bucket b's partials are reduced on st, its
  // all-reduce runs on the communication stream, and Adam on bucket b waits for that bucket
  // only -- Adam of bucket b overlaps the all-reduce of bucket b + 1 (element-wise update)
  cudaStream_t cs = (st == st2) ? st : ctx->cap_stream3;
  const int NB = ctx->ar_buckets;
  const size_t per = ((n + NB - 1) / NB + 255) / 256 * 256;
  int nb = 0;
  for (size_t off = 0; off < n; off += per, ++nb) {
    const size_t len = std::min(per, n - off);
    if (ctx->dw_splits > 1) {
      Stage sg(ctx, st, "reduce_partials");
      CU(launch_reduce_partials_range(ctx->grads + off, len, n, ctx->dw_splits, st));
      ++*nl;
    }
    if (cs != st) {
      cudaEventRecord(ctx->ev_bkt[nb], st);
      cudaStreamWaitEvent(cs, ctx->ev_bkt[nb], 0);
    }
    NC(ncclAllReduce(ctx->grads + off, ctx->grads + off, len, ncclFloat32, ncclSum, ctx->comm, cs));
    if (cs != st) cudaEventRecord(ctx->ev_bkt[crl_ctx::kMaxArBuckets + nb], cs);
  }
  nb = 0;
  for (size_t off = 0; off < n; off += per, ++nb) {
    const size_t len = std::min(per, n - off);
    if (cs != st) cudaStreamWaitEvent(st, ctx->ev_bkt[crl_ctx::kMaxArBuckets + nb], 0);
    Stage sg(ctx, st, "adam");
    CU(launch_adam_ex(ctx->mem.params + off, ctx->grads + off, 1, ctx->mem.adam_m + off, ctx->mem.adam_v + off, len,
                      k.lr, k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay, ctx->adam_t, ctx->skip, ctx->status,
                      shadow ? static_cast<void*>(static_cast<__nv_bfloat16*>(shadow) + off) : nullptr,
                      ctx->num_sms, keep_sum, st));
    ++*nl;
  }
  return CRL_OK;
}

static crl_status enqueue_critic(crl_ctx* ctx, const float* s, const float* a, const float* g,
                                 float* loss_out, float* grads_out, cudaStream_t st,
                                 cudaStream_t st2) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, W = k.world_size, N = ctx->N, D = k.repr_dim;
  const float invN = 1.0f / (float)N;
  // (c_f, c_b): fwd / FlatNCE-fwd (1, 0), bwd / FlatNCE-bwd (0, 1), sym (1, 1); the loss
  // kernels get them negated for FlatNCE (reported value 0, reading A-24)
  const bool bwd_only = k.loss == CRL_LOSS_BWD || k.loss == CRL_LOSS_FLATNCE_BWD;
  const bool fwd_only = k.loss == CRL_LOSS_FWD || k.loss == CRL_LOSS_FLATNCE_FWD;
  const float c_f = bwd_only ? 0.f : 1.f;
  const float c_b = fwd_only ? 0.f : 1.f;
  const float lsgn = (k.loss == CRL_LOSS_FLATNCE_FWD || k.loss == CRL_LOSS_FLATNCE_BWD) ? -1.f : 1.f;
  int nl = 0;
  crl_status rs;
  const bool pair = k.loss >= CRL_LOSS_FB;        // F3 pair / FB losses (W = 1, fp32)
  // A2: encoders forward (phi on st, psi on st2)
  fork(ctx, st, st2);
  rs = enc_forward(ctx, "psi", ctx->psi_plan, g, k.goal_dim, nullptr, 0, 0, ctx->psiX, ctx->psiZ,
                   ctx->psi_out, st2, &nl);
  if (rs != CRL_OK) return rs;
  rs = enc_forward(ctx, "phi", ctx->phi_plan, s, k.obs_dim, a, k.act_dim, k.obs_dim, ctx->phiX,
                   ctx->phiZ, ctx->phi_out, st, &nl);
  if (rs != CRL_OK) return rs;
  join(ctx, st, st2);
  if (ctx->dist) {
    NC(ncclGroupStart());
    NC(ncclAllGather(ctx->phi_out, ctx->phi_g, (size_t)Bl * D, ncclFloat32, ctx->comm, st));
    NC(ncclAllGather(ctx->psi_out, ctx->psi_g, (size_t)Bl * D, ncclFloat32, ctx->comm, st));
    NC(ncclGroupEnd());
  }
  // A3: online row / column logsumexp
  fork(ctx, st, st2);
  { Stage sg(ctx, st2, "lse_col");
    CU(logits_lse_f32(D, k.energy, ctx->psi_out, Bl, ctx->phi_g, N, ctx->lse_col, st2)); ++nl; }
  { Stage sg(ctx, st, "lse_row");
    CU(logits_lse_f32(D, k.energy, ctx->phi_out, Bl, ctx->psi_g, N, ctx->lse_row, st)); ++nl; }
  join(ctx, st, st2);
  if (ctx->dist) {
    NC(ncclGroupStart());
    NC(ncclAllGather(ctx->lse_row, ctx->lse_row_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
    NC(ncclAllGather(ctx->lse_col, ctx->lse_col_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
    NC(ncclGroupEnd());
  }
  if (pair) {
    // d_i = l_ii, per-row pair sums, the loss; then both sides of the gradient
    { Stage sg(ctx, st, "pair_stats");
      CU(launch_pair_diag(ctx->phi_out, ctx->psi_out, Bl, D, k.energy, ctx->pair_d, st)); ++nl;
      CU(logits_pair_stats_f32(D, k.energy, k.loss, ctx->phi_out, Bl, 0, ctx->psi_out, N, ctx->pair_d,
                               ctx->pair_R, ctx->pair_L, st)); ++nl; }
    { Stage sg(ctx, st, "loss");
      CU(launch_pair_loss(ctx->pair_L, ctx->pair_d, ctx->lse_row, Bl, k.loss, invN, k.beta_lse, loss_out,
                          ctx->loss_acc, ctx->skip, ctx->adam_t, ctx->status, st)); ++nl; }
    fork(ctx, st, st2);
    { Stage sg(ctx, st2, "grad_psi");
      CU(logits_pair_grad_f32(D, k.energy, k.loss, 1, ctx->psi_out, Bl, 0, ctx->phi_out, N, ctx->pair_d,
                              ctx->pair_R, ctx->lse_row, k.beta_lse, invN, ctx->dpsi, st2)); ++nl; }
    rs = enc_backward(ctx, "psi", ctx->psi_plan, g, k.goal_dim, nullptr, 0, 0, ctx->psiX, ctx->psiZ,
                      ctx->dpsi, ctx->dz_psi, st2, &nl);
    if (rs != CRL_OK) return rs;
    { Stage sg(ctx, st, "grad_phi");
      CU(logits_pair_grad_f32(D, k.energy, k.loss, 0, ctx->phi_out, Bl, 0, ctx->psi_out, N, ctx->pair_d,
                              ctx->pair_R, ctx->lse_row, k.beta_lse, invN, ctx->dphi, st)); ++nl; }
    rs = enc_backward(ctx, "phi", ctx->phi_plan, s, k.obs_dim, a, k.act_dim, k.obs_dim, ctx->phiX,
                      ctx->phiZ, ctx->dphi, ctx->dz, st, &nl);
    if (rs != CRL_OK) return rs;
    join(ctx, st, st2);
    { Stage sg(ctx, st, "adam");
      CU(launch_adam(ctx->mem.params, ctx->grads, ctx->dw_splits, ctx->mem.adam_m, ctx->mem.adam_v,
                     ctx->sizes.n_params, k.lr, k.adam_b1, k.adam_b2, k.adam_eps, k.weight_decay,
                     ctx->adam_t, ctx->skip, ctx->status, nullptr, ctx->num_sms, st));
      ++nl; }
    if (grads_out)
      CU(cudaMemcpyAsync(grads_out, ctx->grads, ctx->sizes.n_params * 4, cudaMemcpyDeviceToDevice, st));
    ctx->launches = nl;
    return CRL_OK;
  }
  { Stage sg(ctx, st, "loss");
    CU(launch_loss_partial(ctx->phi_out, ctx->psi_out, Bl, D, k.energy, ctx->lse_row, ctx->lse_col,
                           ctx->loss_acc, ctx->loss_part, ctx->loss_ticket, !ctx->dist, invN, lsgn * c_f, lsgn * c_b, k.beta_lse, loss_out, ctx->skip,
                           ctx->adam_t, ctx->status, st));
    ++nl; }
  if (ctx->dist) {
    NC(ncclAllReduce(ctx->loss_acc, ctx->loss_acc, 3, ncclFloat32, ncclSum, ctx->comm, st));
    CU(launch_loss_finalize(ctx->loss_acc, invN, lsgn * c_f, lsgn * c_b, k.beta_lse, loss_out, ctx->skip,
                            ctx->adam_t, ctx->status, st));
    ++nl;
  }
  // A4 (dlogits consumed in-pass) + A5 (encoders backward): phi chain on st, psi on st2
  const int row_off = k.rank * Bl;
  fork(ctx, st, st2);
  { Stage sg(ctx, st2, "grad_psi");
    CU(logits_grad_f32(D, k.energy, ctx->psi_out, Bl, row_off, ctx->phi_g, N, ctx->lse_col,
                       ctx->lse_row_g, c_b, c_f, 0.f, k.beta_lse, invN, ctx->dpsi, st2));
    ++nl; }
  rs = enc_backward(ctx, "psi", ctx->psi_plan, g, k.goal_dim, nullptr, 0, 0, ctx->psiX, ctx->psiZ,
                    ctx->dpsi, ctx->dz_psi, st2, &nl);
  if (rs != CRL_OK) return rs;
  { Stage sg(ctx, st, "grad_phi");
    CU(logits_grad_f32(D, k.energy, ctx->phi_out, Bl, row_off, ctx->psi_g, N, ctx->lse_row,
                       ctx->lse_col_g, c_f, c_b, k.beta_lse, 0.f, invN, ctx->dphi, st));
    ++nl; }
  rs = enc_backward(ctx, "phi", ctx->phi_plan, s, k.obs_dim, a, k.act_dim, k.obs_dim, ctx->phiX,
                    ctx->phiZ, ctx->dphi, ctx->dz, st, &nl);
  if (rs != CRL_OK) return rs;
  join(ctx, st, st2);
  // A6: Adam (sums the split-K partials in the same pass); W > 1: bucketed all-reduce first
  rs = enqueue_allreduce_adam(ctx, st, st2, nullptr, 1, &nl);
  if (rs != CRL_OK) return rs;
  if (grads_out)   // slice 0 holds the reduced pre-Adam gradient after the Adam kernel
    CU(cudaMemcpyAsync(grads_out, ctx->grads, ctx->sizes.n_params * 4, cudaMemcpyDeviceToDevice, st));
  ctx->launches = nl;
  return CRL_OK;
}

// the page-locked host ring of the end-to-end path (host memory; no device allocation)
static bool make_host_ring(crl_ctx* ctx) {
  const crl_config& k = ctx->cfg;
  // slot pitch rounded up to 256 B: every slot base stays 16-byte aligned for the device's
  // 16 B loads whatever B_l * dims is (odd batches with goal_dim 2, e.g.)
  ctx->h_stage_bytes = ((size_t)(reinterpret_cast<char*>(ctx->stage_g) - reinterpret_cast<char*>(ctx->stage_s)) +
                        (size_t)k.batch_local * k.goal_dim * 4 + 255) & ~(size_t)255;
  if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage), ctx->h_stage_bytes * crl_ctx::kHostSlots,
                    cudaHostAllocDefault) != cudaSuccess)
    return false;
  for (int i = 0; i < crl_ctx::kHostSlots; ++i)
    if (cudaEventCreateWithFlags(&ctx->h_ev[i], cudaEventDisableTiming) != cudaSuccess) return false;
  if (cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return false;
  for (int d = 0; d < 2; ++d)
    if (cudaEventCreateWithFlags(&ctx->ev_dcopied[d], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_dfree[d], cudaEventDisableTiming) != cudaSuccess)
      return false;
  return true;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// page-locked host memory the device can address directly (UVA): its device pointer, else null
static const void* mapped_host_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

extern "C" crl_status crl_critic_step(crl_ctx* ctx, const float* s, const float* a, const float* g,
                                      float* loss_out, float* grads_out, void* stream) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  if (!s || !a || !g) return fail(ctx, CRL_EINVAL, "critic_step: NULL batch");
  if (grads_out && !is_device_ptr(grads_out))
    return fail(ctx, CRL_EINVAL, "grads_out must be device memory");
  const crl_config& k = ctx->cfg;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t Bl = k.batch_local;
  // host batch (end-to-end path): copied to the device staging buffers (reading page-locked
  // host memory in place from the input kernel was measured slower: Ant e2e 9.2k -> 7.4k
  // steps/s, the per-element host-link latency); a page-locked host loss is written in place
  // by the loss kernel (CRL_NO_ZERO_COPY: a device-to-host copy instead)
  const bool zc = !std::getenv("CRL_NO_ZERO_COPY");
  int dset = -1;                                          // device staging set of a host batch
  if (ctx->h_stage && !is_device_ptr(s) && !is_device_ptr(a) && !is_device_ptr(g)) {
    // host batch: gathered into a page-locked ring slot laid out like the device staging, then
    // ONE host-to-device copy (three small copies cost three DMA latencies on the timeline)
    const int slot = ctx->h_slot;
    ctx->h_slot = (slot + 1) % crl_ctx::kHostSlots;
    CU(cudaEventSynchronize(ctx->h_ev[slot]));            // the slot's previous copy is done
    char* hb = ctx->h_stage + (size_t)slot * ctx->h_stage_bytes;
    char* d0 = reinterpret_cast<char*>(ctx->stage_s);
    const size_t off_a = reinterpret_cast<char*>(ctx->stage_a) - d0, off_g = reinterpret_cast<char*>(ctx->stage_g) - d0;
    std::memcpy(hb, s, Bl * k.obs_dim * 4);
    std::memcpy(hb + off_a, a, Bl * k.act_dim * 4);
    std::memcpy(hb + off_g, g, Bl * k.goal_dim * 4);
    if (std::getenv("CRL_E2E_PULL")) {
      // the device pulls the slot over the host link with 16 B loads (one small kernel on st,
      // in line with the step; the round-1 design)
      const size_t n16 = (ctx->h_stage_bytes + 15) / 16;
      pull_host_kernel<<<(unsigned)std::min<size_t>((n16 + 255) / 256, (size_t)ctx->num_sms), 256, 0, st>>>(
          reinterpret_cast<uint4*>(ctx->stage_s), reinterpret_cast<const uint4*>(hb), n16);
      CU(cudaGetLastError());
      CU(cudaEventRecord(ctx->h_ev[slot], st));
      s = ctx->stage_s; a = ctx->stage_a; g = ctx->stage_g;
    } else {
      // one DMA copy on the copy engine into the staging set the previous step does NOT read:
      // it overlaps that step's kernels (it waits only for the step two calls back, the last
      // reader of this set); the step waits for its copy
      dset = ctx->d_slot;
      ctx->d_slot ^= 1;
      char* db = dset ? reinterpret_cast<char*>(ctx->stage2) : d0;
      CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_dfree[dset], 0));
      CU(cudaMemcpyAsync(db, hb, ctx->h_stage_bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
      CU(cudaEventRecord(ctx->h_ev[slot], ctx->copy_stream));
      CU(cudaEventRecord(ctx->ev_dcopied[dset], ctx->copy_stream));
      CU(cudaStreamWaitEvent(st, ctx->ev_dcopied[dset], 0));
      s = reinterpret_cast<const float*>(db);
      a = reinterpret_cast<const float*>(db + off_a);
      g = reinterpret_cast<const float*>(db + off_g);
    }
  }
  // the staging set d is free again once this step (its only reader) has run
  auto release_set = [&]() -> crl_status {
    if (dset >= 0) CU(cudaEventRecord(ctx->ev_dfree[dset], st));
    return CRL_OK;
  };
  auto stage_in = [&](const float*& p, float* stage, size_t n) -> crl_status {
    if (is_device_ptr(p)) return CRL_OK;
    CU(cudaMemcpyAsync(stage, p, n * 4, cudaMemcpyHostToDevice, st));
    p = stage;
    return CRL_OK;
  };
  crl_status rs0;
  if ((rs0 = stage_in(s, ctx->stage_s, Bl * k.obs_dim)) != CRL_OK) return rs0;
  if ((rs0 = stage_in(a, ctx->stage_a, Bl * k.act_dim)) != CRL_OK) return rs0;
  if ((rs0 = stage_in(g, ctx->stage_g, Bl * k.goal_dim)) != CRL_OK) return rs0;
  float* loss_dev = ctx->loss_dev;
  bool loss_host = loss_out && !is_device_ptr(loss_out);
  if (loss_out && !loss_host) loss_dev = loss_out;
  if (loss_host && zc)
    if (const void* d = mapped_host_ptr(loss_out)) {
      loss_dev = static_cast<float*>(const_cast<void*>(d));
      loss_host = false;
    }

  if (ctx->prof_on) {                    // eager, event-bracketed launches
    spin_kernel<<<1, 1, 0, st>>>(300000ull);
    crl_status rs = ctx->bf16 ? enqueue_critic_bf16(ctx, s, a, g, loss_dev, grads_out, st, st)
                              : enqueue_critic(ctx, s, a, g, loss_dev, grads_out, st, st);
    if (rs != CRL_OK) return rs;
    if (loss_host) CU(cudaMemcpyAsync(loss_out, loss_dev, 16, cudaMemcpyDeviceToHost, st));
    return release_set();
  }
  GraphKey key{s, a, g, loss_dev, grads_out};
  auto it = ctx->graphs.find(key);
  if (it == ctx->graphs.end() && ctx->graphs.size() >= crl_ctx::kMaxGraphs) {
    // bounded cache: evict the least recently replayed graph (callers that pass fresh
    // tensors every step pay a capture per step, but the cache never grows without bound)
    auto lru = ctx->graph_use.begin();
    for (auto u = ctx->graph_use.begin(); u != ctx->graph_use.end(); ++u)
      if (u->second < lru->second) lru = u;
    const GraphKey old = lru->first;
    cudaGraphExecDestroy(ctx->graphs[old]);
    ctx->graphs.erase(old);
    ctx->graph_launches.erase(old);
    ctx->graph_use.erase(old);
  }
  if (it == ctx->graphs.end()) {
    // capture the schedule once on the private capture stream
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    crl_status rs = ctx->bf16 ? enqueue_critic_bf16(ctx, s, a, g, loss_dev, grads_out, ctx->cap_stream,
                                                    ctx->cap_stream2)
                              : enqueue_critic(ctx, s, a, g, loss_dev, grads_out, ctx->cap_stream,
                                               ctx->cap_stream2);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (rs != CRL_OK) { if (graph) cudaGraphDestroy(graph); return rs; }
    CU(ce);
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CU(ce);
    it = ctx->graphs.emplace(key, exec).first;
    ctx->graph_launches[key] = ctx->launches;
  }
  CU(cudaGraphLaunch(it->second, st));
  ctx->graph_use[key] = ++ctx->use_clock;
  ctx->launches = ctx->graph_launches[key];
  if (loss_host) CU(cudaMemcpyAsync(loss_out, loss_dev, 16, cudaMemcpyDeviceToHost, st));
  return release_set();
}

extern "C" crl_status crl_profile_enable(crl_ctx* ctx, int on) {
  if (!ctx) return fail(ctx, CRL_EINVAL, "ctx is NULL");
  CU(cudaDeviceSynchronize());
  ctx->prof_pending.clear();
  ctx->ev_pool_next = 0;
  ctx->prof_acc.clear();
  ctx->prof_names.clear();
  ctx->prof_on = on != 0;
  return CRL_OK;
}

extern "C" int crl_profile_read(crl_ctx* ctx, int i, char* name_out, int name_cap, double* total_ms,
                                int* count) {
  if (!ctx) return -1;
  if (!ctx->prof_pending.empty()) {
    cudaDeviceSynchronize();
    for (auto& e : ctx->prof_pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e.a, e.b);
      auto& acc = ctx->prof_acc[e.name];
      if (acc.second == 0) ctx->prof_names.push_back(e.name);
      acc.first += ms;
      acc.second += 1;
    }
    ctx->prof_pending.clear();
    ctx->ev_pool_next = 0;
  }
  const int n = (int)ctx->prof_names.size();
  if (i >= 0 && i < n) {
    const std::string& nm = ctx->prof_names[i];
    if (name_out && name_cap > 0) {
      std::strncpy(name_out, nm.c_str(), name_cap - 1);
      name_out[name_cap - 1] = 0;
    }
    if (total_ms) *total_ms = ctx->prof_acc[nm].first;
    if (count) *count = ctx->prof_acc[nm].second;
  }
  return n;
}
