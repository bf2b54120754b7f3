/*
 * crl.h — C ABI of the B200-native contrastive-RL (CRL) critic hot path.
 *
 * Paper: arXiv 2408.11052 "JaxGCRL" (/root/reference/PAPER.md, cited as P:NNN).  The entry
 * points are the four calls north_star names (crl_buffer_insert, crl_relabel_sample,
 * crl_critic_step, crl_actor_loss) plus context management.  Their arguments follow the
 * paper's problem statement: a CMP (S, A, p, p0, gamma) with goals g in S (§3), a
 * batch B of (s_i, a_i, g_i) with g_i from the future of the same trajectory (§3.1
 * P:190-191, §3.2), representations phi(s,a), psi(g) and an energy f over the
 * logits matrix, the critic update with learning rate alpha and logsumexp
 * coefficient beta (Alg. 1), and the actor objective E[f(s, a', g)],
 * a' ~ pi(.|s,g) with a tunable entropy coefficient (Eq. 3).
 *
 * Conventions (apply to every call):
 *  - Every array is row-major and densely packed, fp32 unless stated.
 *  - Device pointers unless a call says "host or device" (then the library inspects the
 *    pointer with cudaPointerGetAttributes and copies host data itself, on `stream`).
 *  - Ownership: the caller allocates and owns every buffer, including the ones passed in
 *    crl_memory at create time; the library keeps non-owning pointers, which must outlive
 *    the context.  The library performs no device allocation after crl_create (crl_create
 *    also allocates a small page-locked HOST ring for host batches of crl_critic_step).
 *  - Asynchrony: calls validate their arguments on the host synchronously and return
 *    CRL_EINVAL / CRL_ESTATE at once; device work is enqueued on `stream` (a cudaStream_t,
 *    passed as void*; NULL = legacy default stream) and the call returns without syncing.
 *    Device-detected faults (non-finite loss or gradient, sampler retry cap) set a device
 *    status word, surfaced by crl_get_status and by the next call on the context.
 *  - Threading: one context per (process, GPU); calls on one context are not re-entrant.
 *  - Multi-GPU: each rank passes rank-local pointers, its `rank` and `world_size`;
 *    returned losses and gradients are global (all-reduced) values.
 *  - Errors never cross the ABI as exceptions; crl_last_error() gives a message.
 */
#ifndef CRL_H_
#define CRL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CRL_ABI_VERSION 3   /* 2: crl_config gained layernorm, random_goal_alpha;
                               3: random goals go to the actor's goals only (crl_relabel_sample_mixed) */

#if defined(__GNUC__)
#define CRL_API __attribute__((visibility("default")))
#else
#define CRL_API
#endif

typedef enum {
  CRL_OK = 0,
  CRL_EINVAL = 1,        /* bad argument: dims, B < 2, misaligned or NULL pointer          */
  CRL_ESTATE = 2,        /* call order, or the buffer holds < 2 slots per env              */
  CRL_ECUDA = 3,         /* a CUDA runtime call failed                                     */
  CRL_ENCCL = 4,         /* an NCCL call failed                                            */
  CRL_ENONFINITE = 5,    /* device saw a NaN/Inf loss or gradient (Adam step skipped)      */
  CRL_ESAMPLER = 6,      /* a row found no valid start in 64 attempts (reading A-10)       */
  CRL_EUNSUPPORTED = 7   /* configuration not supported by this build                      */
} crl_status;

typedef enum {
  CRL_ENERGY_L2 = 0, CRL_ENERGY_DOT = 1, CRL_ENERGY_COS = 2, CRL_ENERGY_L1 = 3, CRL_ENERGY_L2SQ = 4
} crl_energy;
/* L2: f = -||phi - psi||_2 (App. A.2, sign per reading A-01)
 * DOT: f = <phi, psi>;  COS: f = <phi,psi>/(||phi|| ||psi||)
 * L1: f = -||phi - psi||_1 (derivative 0 at ties, reading A-33);
 * L2SQ: f = -||phi - psi||_2^2 ("L2 w/o sqrt").  L1 and L2SQ run on
 * the fp32 path (critic and actor); L2SQ also on the bf16 tensor-core path (the same
 * contraction as L2).  A bf16 context with L1 is CRL_EUNSUPPORTED. */
typedef enum {
  CRL_LOSS_FWD = 0, CRL_LOSS_BWD = 1, CRL_LOSS_SYM = 2, CRL_LOSS_FLATNCE_FWD = 3, CRL_LOSS_FLATNCE_BWD = 4,
  CRL_LOSS_FB = 5, CRL_LOSS_DPO = 6, CRL_LOSS_IPO = 7, CRL_LOSS_SPPO = 8
} crl_loss;
/* InfoNCE forward / backward / symmetric = fwd + bwd (App. A.2).
 * FlatNCE fwd / bwd: L = (1/N) sum_i log(S_i / sg[S_i]),
 * S_i = sum_j exp(l_ij - l_ii) (sign per reading A-24): its value is 0 and its gradient is
 * exactly the InfoNCE fwd / bwd gradient, so it runs the InfoNCE kernels and reports
 * L_fwd = L_bwd = 0, total = the logsumexp penalty.  Both precisions.
 * FB, DPO, IPO, SPPO (readings A-03 mean over the N positives,
 * A-34 j ranges as printed): no logsumexp in the objective (the row-LSE penalty still
 * applies); loss_out = (L_pair, 0, penalty, total).  fp32 and world_size 1 only, else
 * CRL_EUNSUPPORTED at create. */
typedef enum { CRL_ACT_SILU = 0, CRL_ACT_RELU = 1 } crl_activation;
typedef enum { CRL_FP32 = 0, CRL_BF16 = 1 } crl_precision;
/* FP32: SIMT fp32 arithmetic end to end.  BF16: bf16 GEMM operands on the tcgen05 tensor
 * cores with fp32 accumulation, fp32 statistics / loss / gradients / optimiser state. */

typedef struct {
  /* spaces (§3): g = obs[goal_offset : goal_offset + goal_dim] (reading A-12) */
  int obs_dim, act_dim, goal_dim, goal_offset;
  /* replay buffer: E_l envs on this rank, capacity T slots per env (Table 2) */
  int n_envs_local, capacity;
  double gamma;                    /* discounting, 0 <= gamma < 1 (Table 2)          */
  /* encoders phi([s||a]) and psi(g): depth hidden layers of `width`, output repr_dim
   * (Table 2; §5.4); activation per reading A-13                     */
  int depth, width, repr_dim, activation;
  int energy, loss;                /* crl_energy, crl_loss                                 */
  float beta_lse;                  /* logsumexp penalty coefficient         */
  float lr, adam_b1, adam_b2, adam_eps, weight_decay;  /* critic Adam (A-15)        */
  int precision;                   /* crl_precision                                        */
  int batch_local, world_size, rank; /* global batch N = batch_local * world_size          */
  int actor_depth, actor_width;    /* actor MLP [s||g] -> (mu, log sigma)          */
  float lr_actor;                  /* policy_lr                                    */
  int layernorm;                   /* 1: LayerNorm before every hidden activation (F2;
                                      §5.4, reading A-35: per-row over features,
                                      gain + shift, eps 1e-6).  Parameters per hidden layer:
                                      W, b, gamma[out], beta[out].  fp32 path only (bf16 ->
                                      CRL_EUNSUPPORTED); the actor has no LayerNorm. */
  float random_goal_alpha;         /* F4 random-goal mixing in [0, 1] (App. C P:951-964,
                                      reading A-36): the fraction of the ACTOR's goals
                                      (crl_relabel_sample_mixed g_actor) that is the goal
                                      slice of a uniformly random stored state instead of the
                                      hindsight goal; the critic's g is never mixed; 0 = off */
} crl_config;

typedef struct {
  size_t n_params;        /* critic params (phi then psi), floats                          */
  size_t n_actor_params;  /* actor params, floats (0 if actor_depth == 0)                  */
  size_t buffer_bytes;    /* replay rings + per-slot episode metadata + offset table       */
  size_t scratch_bytes;   /* activations, statistics, gradients, bf16 operand shadows      */
} crl_sizes;

typedef struct {
  /* Flat fp32 parameters: for phi then psi, for each layer W[in][out] then b[out]
   * (layers: depth hidden, then the output layer).  Initial values are the caller's. */
  float* params;          /* [n_params]                                                    */
  float* adam_m;          /* [n_params], zero-initialised by the caller                    */
  float* adam_v;          /* [n_params], zero-initialised by the caller                    */
  float* actor_params;    /* [n_actor_params] or NULL (same per-layer layout)              */
  float* actor_adam_m;    /* [n_actor_params] or NULL                                      */
  float* actor_adam_v;    /* [n_actor_params] or NULL                                      */
  void* buffer;           /* [buffer_bytes], 256-byte aligned                              */
  void* scratch;          /* [scratch_bytes], 256-byte aligned                             */
} crl_memory;

typedef struct crl_ctx crl_ctx;

/* Sizes of the caller-owned regions for `cfg`.  Pure host computation; no GPU needed. */
CRL_API crl_status crl_workspace_size(const crl_config* cfg, crl_sizes* out);

/* Create a context on the current CUDA device.  `nccl_unique_id` points to the 128-byte
 * ncclUniqueId obtained by rank 0 with crl_nccl_unique_id and broadcast by the caller
 * (NULL when world_size == 1).  Uploads the host-built geometric offset table (contract
 * C1: G[k] = gamma^k by repeated fp64 multiplication, Q[k] = floor((1 - G[k]) 2^64)) into
 * `buffer` and zeroes the episode metadata.  Synchronises the device once. */
CRL_API crl_status crl_create(const crl_config* cfg, const crl_memory* mem, const void* nccl_unique_id,
                      crl_ctx** out);
CRL_API crl_status crl_destroy(crl_ctx* ctx);

/* rank 0: write a fresh 128-byte NCCL unique id to `out128` (host memory). */
CRL_API crl_status crl_nccl_unique_id(void* out128);

/* A0 — append U steps of every local env, in lock-step (Alg. 1).
 *   obs  [U][E_l][obs_dim]  device, fp32
 *   act  [U][E_l][act_dim]  device, fp32
 *   done [U][E_l]           device, uint8: 1 = the transition taken at that step ended the
 *                           episode; the next step of that env starts a new one
 * Step u of env e lands at absolute index n_ins + u (n_ins = steps inserted so far) in ring
 * slot (n_ins + u) mod T; the oldest steps are overwritten once the ring is full.  Per-slot
 * episode-end metadata is back-filled (amortised O(1) per step).  One kernel; no sync. */
CRL_API crl_status crl_buffer_insert(crl_ctx* ctx, const float* obs, const float* act,
                             const uint8_t* done, int U, void* stream);

/* A1 — hindsight relabel sample of batch_local rows (contract C1; P:165-169, P:190-191,
 * P:219, Alg. 1).  Row r (global row rho = rank*batch_local + r), attempt a:
 *   (x0..x3) = Philox4x32-10(ctr = (rho, a, lo32(step), hi32(step)), key = (lo32(seed), hi32(seed)))
 *   e = (x0 * E_l) >> 32,  tau = tau_old + ((x1 * n) >> 32)
 *   L = (first tau' >= tau with done = 1, capped at tau_new) - tau;  accept if L >= 1
 *   k = min{k in [1,L] : Q[k] > ((x2<<32|x3) * Q[L]) >> 64}
 * Outputs (device): s[B_l][obs_dim] = obs(e, tau), a[B_l][act_dim] = act(e, tau),
 *   g[B_l][goal_dim] = obs(e, tau+k)[goal_offset:], idx[B_l][3] int64 = (rank*E_l + e, tau,
 *   tau+k) in absolute steps (idx may be NULL).  Integer-only device arithmetic: the result
 *   is bit-exact w.r.t. the oracle.  CRL_ESTATE if fewer than 2 slots are stored. */
CRL_API crl_status crl_relabel_sample(crl_ctx* ctx, uint64_t seed, uint64_t step, float* s, float* a,
                              float* g, int64_t* idx, void* stream);

/* F4 — bulk sampling for several updates in one launch (Alg. 1 P:1044-1046 runs num_updates
 * gradient steps per collection round).  Output row u*batch_local + r is
 * exactly row r of crl_relabel_sample(seed, step0 + u): s[n_updates*B_l][obs_dim],
 * a[n_updates*B_l][act_dim], g[n_updates*B_l][goal_dim], idx[n_updates*B_l][3] (idx may be
 * NULL), all device.  CRL_EINVAL if n_updates < 1 or n_updates * batch_local > 2^30. */
CRL_API crl_status crl_relabel_sample_bulk(crl_ctx* ctx, uint64_t seed, uint64_t step0, int n_updates,
                                           float* s, float* a, float* g, int64_t* idx, void* stream);

/* F4 — bulk sampling plus the actor's goals under random-goal mixing (App. C P:951-964 mixes
 * uniformly random goals into the POLICY objective; reading A-36).  s, a, g, idx exactly as
 * crl_relabel_sample_bulk (g = hindsight goals: the critic's batch).  g_actor
 * [n_updates*B_l][goal_dim] (device, required): row r is g's row unless Philox draw
 * (rho, 64, step) has y0 < floor(random_goal_alpha 2^32), in which case it is the goal slice
 * of the stored state (env (y1 E_l) >> 32, slot tau_old + ((y2 n) >> 32)).  Bit-exact
 * w.r.t. oracle/replay.py random_goal_mix.  Errors as crl_relabel_sample_bulk; CRL_EINVAL
 * for a NULL g_actor. */
CRL_API crl_status crl_relabel_sample_mixed(crl_ctx* ctx, uint64_t seed, uint64_t step0, int n_updates,
                                            float* s, float* a, float* g, float* g_actor, int64_t* idx,
                                            void* stream);

/* A2-A6 — one critic update (Alg. 1) on the batch (s, a, g):
 *   phi = phi_enc([s||a]), psi = psi_enc(g); l_ij = f(phi_i, psi_j) over the GLOBAL batch
 *   (global negatives, reading A-21); L = c_f L_fwd + c_b L_bwd + beta mean_i LSE_i^2
 *   (readings A-02..A-05), computed with online row/column logsumexps so the N x N logits
 *   are never stored; dL/dl consumed in-pass; reverse mode through both encoders; gradients
 *   all-reduced across ranks; one fused bias-corrected Adam step on `params` (A-15).
 *   s [B_l][obs_dim], a [B_l][act_dim], g [B_l][goal_dim]: host or device.
 *   loss_out: float[4] = (L_fwd, L_bwd, penalty, total), host or device, may be NULL
 *   (page-locked host memory is written in place by the loss kernel; other host memory by a
 *   device-to-host copy on `stream`).
 *   grads_out: device float[n_params] pre-Adam global gradients, or NULL.
 * The device sequence is captured once per distinct pointer tuple into a CUDA graph and
 * replayed.  If the gradient or loss is non-finite the Adam step is skipped and the status
 * word is set to CRL_ENONFINITE. */
CRL_API crl_status crl_critic_step(crl_ctx* ctx, const float* s, const float* a, const float* g,
                           float* loss_out, float* grads_out, void* stream);

/* Actor loss (Eq. 3; entropy coefficient P:313; alpha = 0 random goals, App. C):
 *   [mu, log_sigma] = pi([s||g]) with log_sigma clipped to [-5, 2]; u = mu + sigma*eps;
 *   a' = tanh(u); log pi = sum(-eps^2/2 - log sigma - log(2 pi)/2) - sum log(1 - a'^2 + 1e-6);
 *   L = mean_i(alpha_ent log pi_i - f(phi([s_i||a'_i]), psi(g_i)))   (critic frozen).
 *   s [B_l][obs_dim], g [B_l][goal_dim], eps [B_l][act_dim] ~ N(0,1): device.
 *   loss_out: device float[1] or NULL; actor_grads_out: device float[n_actor_params] or NULL;
 *   apply_adam != 0 applies one Adam step (lr_actor, adam_b1/b2/eps, weight_decay) to
 *   actor_params; the step is skipped and CRL_ENONFINITE raised if the loss is non-finite.
 * Multi-GPU: the loss is the global mean and the gradients are all-reduced (sum of 1/N terms).
 * fp32 throughout (the critic's fp32 master parameters); the schedule is captured once per
 * (s, g, eps, loss_out, actor_grads_out, apply_adam) into a CUDA graph and replayed on
 * `stream` (alpha_ent is written to device memory first, so any alpha reuses the graph).
 * CRL_EUNSUPPORTED if the context was created without an actor (actor_depth = 0). */
CRL_API crl_status crl_actor_loss(crl_ctx* ctx, const float* s, const float* g, const float* eps,
                          float alpha_ent, float* loss_out, float* actor_grads_out,
                          int apply_adam, void* stream);

/* Entropy coefficient update ("a tuneable entropy coefficient"; the paper gives no
 * rule, reading A-32 takes SAC's automatic tuning):
 *   L_alpha = alpha * (-mean_i log pi_i - target_entropy),  alpha = exp(*log_alpha),
 * one Adam step on log_alpha (context adam_b1/b2/eps, no weight decay, own step counter)
 * with gradient dL_alpha/dlog_alpha = L_alpha; mean log pi is the global mean from the last
 * crl_actor_loss on this context (CRL_ESTATE if there was none).
 *   log_alpha: device float[1], read and updated in place.  alpha_out: device float[1] or
 *   NULL (exp of the new log_alpha).  loss_out: device float[1] or NULL (L_alpha).
 * A non-finite L_alpha leaves log_alpha unchanged and sets CRL_ENONFINITE in the status word.
 * Launched on `stream` after the actor loss (stream order carries the dependency).
 * CRL_EUNSUPPORTED without an actor; CRL_EINVAL for NULL log_alpha, lr <= 0 or a
 * non-finite target. */
CRL_API crl_status crl_entropy_update(crl_ctx* ctx, float target_entropy, float lr, float* log_alpha,
                                      float* alpha_out, float* loss_out, void* stream);

/* Device status word: CRL_OK or the first device-detected fault since the last reset.
 * sync != 0 synchronises the device first; reset clears it. */
CRL_API crl_status crl_get_status(crl_ctx* ctx, int sync, int reset);
CRL_API const char* crl_last_error(const crl_ctx* ctx);   /* ctx may be NULL (global last error) */

/* Debug taps (parity tests): device pointer and element count of an internal fp32 tensor
 * written by the last crl_critic_step: "phi" [B_l][D], "psi" [B_l][D], "lse_row" [B_l],
 * "lse_col" [B_l] (this rank's columns), "dphi", "dpsi" [B_l][D], "grads" [n_params] (the
 * reduced pre-Adam gradient on the bf16 path only when the step was given grads_out: without
 * it the split-K partials are summed inside the Adam kernel and not written back).
 * Valid until the next call on the context. */
CRL_API crl_status crl_debug_tensor(crl_ctx* ctx, const char* name, const float** ptr, size_t* count);

/* Profiling mode (measurement only, bench.py roofline): while enabled, crl_critic_step
 * launches its schedule eagerly instead of replaying the graph and brackets every kernel
 * with CUDA events on `stream`; crl_relabel_sample does the same.  Enabling / disabling
 * synchronises the device and clears the per-stage totals. */
CRL_API crl_status crl_profile_enable(crl_ctx* ctx, int on);
/* Number of distinct stages recorded so far (synchronises on first read after new launches);
 * for 0 <= i < n also writes stage i's name (NUL-terminated, truncated to name_cap), its
 * summed event time in ms and its launch count. */
CRL_API int crl_profile_read(crl_ctx* ctx, int i, char* name_out, int name_cap, double* total_ms,
                             int* count);

/* Kernel launches enqueued by the last call on the context (bench `gpu_launches`). */
CRL_API int crl_last_launch_count(const crl_ctx* ctx);

CRL_API int crl_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CRL_H_ */
