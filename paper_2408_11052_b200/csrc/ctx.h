// ctx.h — internal definition of crl_ctx and the host-side helpers shared by the C ABI
// (crl_api.cu) and the BF16 tensor-core schedule (step_bf16.cu).  Not part of the ABI.
#pragma once
#include <cstdlib>
#include "common.cuh"
#include "tc_common.cuh"
#include "tc_cchain.h"
#include "tc_chain.h"
#include "tc_dwg.h"
#include "tc_pdw.h"
#include "tc_pgemm.h"
#include "tc_grad2.h"

#include <nccl.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

namespace crl {
cudaError_t launch_buffer_insert(const float*, const float*, const uint8_t*, int, int, int, int, int,
                                 int, int, uint32_t, float*, float*, uint32_t*, uint32_t*,
                                 cudaStream_t);
cudaError_t launch_relabel_sample(int, int, int, int, int, int, int, int, int, int, int, uint32_t,
                                  uint32_t, uint64_t, uint64_t, double, uint64_t, const float*, const float*,
                                  const uint32_t*, const uint64_t*, float*, float*, float*,
                                  float*, int64_t*, int*, cudaStream_t);
cudaError_t mlp_forward_layer_f32(int, int, int, const float*, int, const float*, int, int,
                                  const float*, const float*, float*, float*, int, cudaStream_t);
cudaError_t mlp_backward_dx_f32(int, int, int, const float*, const float*, const float*, float*,
                                int, cudaStream_t);
cudaError_t mlp_backward_dw_f32(int, int, int, const float*, int, const float*, int, int,
                                const float*, float*, float*, int, size_t, cudaStream_t);
int dw_splits_for(int Bn);
inline bool force_dist() { return std::getenv("CRL_FORCE_DIST") != nullptr; }
void gemm_set_num_sms(int n);
void logits_set_num_sms(int n);
cudaError_t launch_reduce_partials(float*, size_t, int, cudaStream_t);
cudaError_t launch_reduce_partials_range(float*, size_t, size_t, int, cudaStream_t);
// W > 1: split-K partials reduced, gradient all-reduced in buckets on a communication stream,
// Adam per bucket on st as soon as its bucket is reduced; W = 1: plain Adam
crl_status enqueue_allreduce_adam(crl_ctx* ctx, cudaStream_t st, cudaStream_t st2, void* shadow, int keep_sum,
                                  int* nl);
bool logits_simt_supports(int D);
cudaError_t logits_lse_f32(int, int, const float*, int, const float*, int, float*, cudaStream_t);
cudaError_t logits_grad_f32(int, int, const float*, int, int, const float*, int, const float*,
                            const float*, float, float, float, float, float, float*, cudaStream_t);
cudaError_t launch_loss_partial(const float*, const float*, int, int, int, const float*,
                                const float*, float*, float*, unsigned*, int, float, float, float,
                                float, float*, int*, int*, int*, cudaStream_t);
int loss_partial_blocks(int Bl);
bool ln_bf16_supports(int N);
cudaError_t launch_ln_fwd_bf16(int, int, const __nv_bfloat16*, const float*, const float*, int, __nv_bfloat16*,
                               __nv_bfloat16*, float*, float*, cudaStream_t);
cudaError_t launch_ln_bwd_bf16(int, int, __nv_bfloat16*, const __nv_bfloat16*, const float*, const float*, const float*,
                               float*, int, float*, float*, int, size_t, cudaStream_t);
cudaError_t launch_ln_fwd(int, int, const float*, const float*, const float*, int, float*, float*, float*, float*,
                          cudaStream_t);
cudaError_t launch_ln_bwd(int, int, float*, const float*, const float*, const float*, const float*, float*, float*,
                          int, size_t, cudaStream_t);
cudaError_t launch_pair_diag(const float*, const float*, int, int, int, float*, cudaStream_t);
cudaError_t launch_pair_loss(const float*, const float*, const float*, int, int, float, float, float*, float*, int*,
                             int*, int*, cudaStream_t);
cudaError_t logits_pair_stats_f32(int, int, int, const float*, int, int, const float*, int, const float*, float*,
                                  float*, cudaStream_t);
cudaError_t logits_pair_grad_f32(int, int, int, int, const float*, int, int, const float*, int, const float*,
                                 const float*, const float*, float, float, float*, cudaStream_t);
cudaError_t launch_loss_finalize(const float*, float, float, float, float, float*, int*, int*,
                                 int*, cudaStream_t);
cudaError_t launch_adam(float*, float*, int, float*, float*, size_t, float, float, float, float,
                        float, const int*, const int*, int*, void*, int, cudaStream_t);
cudaError_t launch_adam_ex(float*, float*, int, float*, float*, size_t, float, float, float, float,
                           float, const int*, const int*, int*, void*, int, int, cudaStream_t);
cudaError_t launch_adam_range(float* p, float* g, int S, size_t gs, float* m, float* v, size_t n, float lr,
                              float b1, float b2, float eps, float wd, const int* adam_t, const int* skip,
                              int* status, void* shadow_bf16, int num_sms, int keep_sum, cudaStream_t st);
namespace tc {
bool tc_logits_supports(int D);
int tc_logits_splits(int Na, int Nb, int D, int num_sms);
bool tc_stats_supports(int D, int energy);
int tc_stats_splits(int Na, int Nb, int num_sms);
bool tc_gradf_supports(int D, int energy);
int tc_gradf_splits(int Na, int Nb, int num_sms);
}  // namespace tc
using tc::tc_gradf_supports;
using tc::tc_gradf_splits;
using tc::tc_logits_supports;
using tc::tc_logits_splits;
using tc::tc_stats_supports;
using tc::tc_stats_splits;
}  // namespace crl

using namespace crl;

extern thread_local std::string g_last_error;

// ----------------------------------------------------------------------------------------
// workspace carving (shared by crl_workspace_size and crl_create)
// ----------------------------------------------------------------------------------------
struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct GraphKey {
  const void *s, *a, *g, *loss, *grads;
  bool operator<(const GraphKey& o) const {
    return std::tie(s, a, g, loss, grads) < std::tie(o.s, o.a, o.g, o.loss, o.grads);
  }
};

struct ActorKey {
  const void *s, *g, *eps, *loss, *grads;
  int adam;
  bool operator<(const ActorKey& o) const {
    return std::tie(s, g, eps, loss, grads, adam) < std::tie(o.s, o.g, o.eps, o.loss, o.grads, o.adam);
  }
};

struct crl_ctx {
  crl_config cfg{};
  crl_sizes sizes{};
  crl_memory mem{};
  EncoderPlan phi_plan{}, psi_plan{};
  int N = 0;
  // replay buffer
  float* obs_ring = nullptr; float* act_ring = nullptr;
  uint32_t* ep_end = nullptr; uint32_t* open_start = nullptr; uint64_t* qtab = nullptr;
  int obs_stride = 0, act_stride = 0;
  uint64_t n_ins = 0;
  // scratch
  float* grads = nullptr;             // [dw_splits][n_params] split-K partials, slice 0 = sum
  int dw_splits = 1;
  float* phiX[CRL_MAX_LAYERS] = {}; float* phiZ[CRL_MAX_LAYERS] = {};
  // F2 LayerNorm: Y = LN(Z) (post-norm, pre-activation), row mean and 1/std per hidden layer
  float* phiY[CRL_MAX_LAYERS] = {}; float* psiY[CRL_MAX_LAYERS] = {};
  float* phiMu[CRL_MAX_LAYERS] = {}; float* psiMu[CRL_MAX_LAYERS] = {};
  float* phiRs[CRL_MAX_LAYERS] = {}; float* psiRs[CRL_MAX_LAYERS] = {};
  float* psiX[CRL_MAX_LAYERS] = {}; float* psiZ[CRL_MAX_LAYERS] = {};
  float *phi_out = nullptr, *psi_out = nullptr, *phi_g = nullptr, *psi_g = nullptr;
  float *lse_row = nullptr, *lse_col = nullptr, *lse_row_g = nullptr, *lse_col_g = nullptr;
  float *dphi = nullptr, *dpsi = nullptr, *dz[2] = {nullptr, nullptr}, *dz_psi[2] = {nullptr, nullptr};
  float *loss_acc = nullptr, *loss_dev = nullptr, *loss_part = nullptr;
  float *pair_d = nullptr, *pair_R = nullptr, *pair_L = nullptr;   // F3 pair losses [B_l]
  unsigned* loss_ticket = nullptr;
  int *status = nullptr, *adam_t = nullptr, *skip = nullptr;
  float *stage_s = nullptr, *stage_a = nullptr, *stage_g = nullptr;
  // end-to-end path: page-locked host ring mirroring [stage_s .. stage_g] so a host batch
  // travels in ONE host-to-device copy (slots reused once their copy has completed)
  static constexpr int kHostSlots = 4;
  char* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  int h_slot = 0;
  cudaEvent_t h_ev[kHostSlots] = {};
  // two device staging sets (stage_s.. and stage2 with the same layout) alternate between host
  // batches: step i + 1's host-to-device copy runs on the copy engine (copy_stream) while step i
  // computes; ev_dcopied[d]: set d landed, ev_dfree[d]: the step that read set d finished
  float* stage2 = nullptr;
  int d_slot = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_dcopied[2] = {}, ev_dfree[2] = {};
  // runtime
  cudaStream_t cap_stream = nullptr, cap_stream2 = nullptr, cap_stream3 = nullptr, cap_stream4 = nullptr;
  cudaStream_t cap_body = nullptr;        // captures the bodies of conditional graph nodes
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_side = nullptr;
  // C4 bucketed gradient all-reduce (W > 1): [2][kMaxArBuckets] events (partials reduced, all-reduced)
  static constexpr int kMaxArBuckets = 8;
  int ar_buckets = 1;
  std::vector<cudaEvent_t> ev_bkt;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int> graph_launches;     // kernels per replay of each cached graph
  std::map<GraphKey, uint64_t> graph_use;     // last replay (LRU eviction beyond kMaxGraphs)
  uint64_t use_clock = 0;
  static constexpr size_t kMaxGraphs = 16;
  ncclComm_t comm = nullptr;
  int num_sms = 148;
  int launches = 0;
  std::string err;
  // profiling mode (eager launches bracketed by CUDA events, per-stage totals)
  bool prof_on = false;
  struct ProfEv { std::string name; cudaEvent_t a, b; };
  std::vector<ProfEv> prof_pending;
  std::vector<std::string> prof_names;
  std::map<std::string, std::pair<double, int>> prof_acc;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_pool_next = 0;
  // ---------------- BF16 tensor-core path (precision == CRL_BF16)
  bool bf16 = false;
  // the data-parallel code path (collectives, global gather buffers, two-call logits): world_size > 1,
  // or CRL_FORCE_DIST=1 at world_size 1 (a one-rank NCCL communicator: the multi-GPU
  // schedule exercised on one GPU, tests/test_gpu_parity.py::test_critic_step_forced_dist_path)
  bool dist = false;
  float* st_colsum = nullptr;                           // W > 1: this rank's column sums of e^l [N]
  __nv_bfloat16* wshadow = nullptr;           // bf16 copy of params (written by Adam)
  __nv_bfloat16 *x0_phi = nullptr, *x0_psi = nullptr;   // [B][ld0_phi], [B][ld0_psi]
  int ld0_phi = 0, ld0_psi = 0;
  __nv_bfloat16* phiXb[CRL_MAX_LAYERS] = {}; __nv_bfloat16* phiZb[CRL_MAX_LAYERS] = {};
  __nv_bfloat16* psiXb[CRL_MAX_LAYERS] = {}; __nv_bfloat16* psiZb[CRL_MAX_LAYERS] = {};
  __nv_bfloat16 *phi_outb = nullptr, *psi_outb = nullptr;   // Y in bf16 (logits operands)
  __nv_bfloat16 *dphib = nullptr, *dpsib = nullptr;         // dY in bf16
  // dZ_l of every hidden layer has its own buffer: db_l is reduced on a side stream, so a
  // ping-pong buffer would be overwritten while the side stream still reads it
  __nv_bfloat16* dzb_phi[CRL_MAX_LAYERS] = {};
  __nv_bfloat16* phiYb[CRL_MAX_LAYERS] = {}; __nv_bfloat16* psiYb[CRL_MAX_LAYERS] = {};   // LN (bf16): Y = LN(Z)
  int ln_nblk = 0;
  float* ln_part_phi = nullptr; float* ln_part_psi = nullptr;            // LN (bf16): dgamma / dbeta partials
  __nv_bfloat16* dzb_psi[CRL_MAX_LAYERS] = {};
  struct TcLayer {
    CUtensorMap fwdA, fwdB, dwA, dwB, dxA, dxB;
    int bn_fwd = 64, bn_dw = 64, bn_dx = 64;
    const __nv_bfloat16* dz = nullptr;   // dZ_l (bf16) consumed by this layer's backward
    __nv_bfloat16* dzprev = nullptr;     // dZ_{l-1} written by this layer's dX GEMM
    // wide layers: the persistent CTA-pair GEMM (tc_pgemm.cu) for the forward / dX products
    bool pg_fwd = false, pg_dx = false;
    tc::PgemmMaps pgf{}, pgd{};
  };
  std::vector<TcLayer> tc_phi, tc_psi;
  // tensor-core logits stage (bf16 path with N >= kTcLogitsMinN)
  bool tc_logits = false;
  int lg_splits = 1;
  __nv_bfloat16 *phi_outb_g = nullptr, *psi_outb_g = nullptr;   // global (gathered) bf16 reps
  float *stat_phi = nullptr, *stat_psi = nullptr;               // [N + pad] |x|^2 or 1/|x|
  float *fac_row = nullptr, *fac_col = nullptr;                 // 2^(-LSE log2e) per local row / column
  float *fac_row_g = nullptr, *fac_col_g = nullptr;             // gathered (aliases when W = 1)
  int* fac_ok = nullptr;                                        // all factors normal this step
  // fused per-row-block MLP chains (bf16 path, width <= 256): one launch for both encoders'
  // forward, one for both encoders' dX chain
  bool use_chain = false;
  tc::ChainMaps chain_fwd[2], chain_bwd[2];
  tc::ChainParams chain_fwd_p{}, chain_bwd_p{};
  float *lg_part_m = nullptr, *lg_part_s = nullptr, *lg_part_da = nullptr, *lg_part_rs = nullptr;
  int* lg_ticket = nullptr;        // [2][row blocks] in-kernel LSE merge tickets (zeroed at create)
  CUtensorMap lg_row_A, lg_row_B, lg_col_A, lg_col_B;
  // fused row + column statistics in one pass (tc_stats.cu; W = 1, L2 / cos, D <= 128)
  bool use_stats = false;
  int st_splits = 1, st_ldc = 0;
  float *st_part_rs = nullptr;                // [st_splits][B_l] row sums
  float *st_colpart = nullptr;                // [row blocks][st_ldc] column sums
  int* st_bad = nullptr;                      // set by the merge: the exact online-max path runs
  CUtensorMap st_A, st_B;                     // its operand maps (A, B boxes {64, 128})
  // both gradient sides in one pass (tc_gradf.cu; W = 1, L2 / dot, D = 64)
  bool use_gradf = false;
  int gf_splits = 1;
  float *gf_part_da = nullptr, *gf_part_rs = nullptr;   // row side per split
  float *gf_acc = nullptr, *gf_cs = nullptr;            // column side [N][64], [N] (reductions)
  size_t gf_acc_bytes = 0;
  CUtensorMap gf_map;
  // both gradient sides in one persistent launch at D = 256 (tc_grad2.cu)
  bool use_grad2 = false;
  int g2_grid = 0;
  float *g2_part_da = nullptr, *g2_part_rs = nullptr;   // [2 sides][2 slots][B_l][D], [2][2][B_l]
  unsigned char* g2_flags = nullptr;                    // [2 sides][row blocks] slot-1 flags
  CUtensorMap g2_B0, g2_B1;                             // B operands (box {64, 128}): Psi_g, Phi_g
  bool g2_pair = false;                                 // CTA-pair variant (tc_grad2p)
  CUtensorMap g2_S0, g2_S1;                             // pair: S parts (box {64, 64}): Psi_g, Phi_g
  CUtensorMap g2_A0, g2_A1;        // CTA-pair gradient pass: local Phi / Psi rows, box {64, 128}
  // W = 1, symmetric energies (L2, L2^2, dot): the pair pass does side 0 only and stores W;
  // dPsi = W^T Phi and the column sums of W come from one pair GEMM (tc_pdw.cu pdw_add_gemm)
  bool g2_wsym = false;
  __nv_bfloat16* g2_W = nullptr;   // [B_l][N] bf16
  float* g2_cs = nullptr;          // [2 slices][N] column sums of W
  CUtensorMap g2_Wmap;             // W, box {64, 128} (the pass's TMA stores)
  tc::PdwParams pdw_g;             // the W^T Phi GEMM
  // all weight / bias gradients of both encoders in one grouped launch (tc_dwg.cu)
  bool use_dwg = false;
  tc::DwgParams dwg;
  bool use_pdw = false;            // wide encoders: dW / db on CTA pairs (tc_pdw.cu) instead of tc_dwg
  tc::PdwParams pdw;
  // W = 1: phi's dW / db (pdw) and psi's (pdw_psi) as two launches on two streams, each
  // followed by Adam over its encoder's parameters (the first Adam overlaps the other dW tail)
  bool pdw_split = false;
  tc::PdwParams pdw_psi;
  // cluster-split MLP chains for small batches (tc_cchain.cu): one launch per direction
  bool use_cchain = false;
  tc::CChainMaps cchain_fwd[2], cchain_bwd[2];
  tc::CChainParams cchain_fwd_p{}, cchain_bwd_p{};
  // ---------------- actor objective (crl_actor_loss, actor.cu): fp32 SIMT, critic frozen
  bool has_actor = false;
  EncoderPlan actor_plan{};
  float* aX[CRL_MAX_LAYERS] = {}; float* aZ[CRL_MAX_LAYERS] = {};      // actor activations
  float *a_out = nullptr;                  // [B_l][2 act]: (mu, log sigma raw)
  float *a_new = nullptr;                  // [B_l][act]: a' = tanh(mu + sigma eps)
  float *a_logpi = nullptr, *a_rowloss = nullptr;   // [B_l]
  float *a_dout = nullptr, *a_da = nullptr;         // [B_l][2 act], [B_l][act]
  float* a_dz[2] = {nullptr, nullptr};     // actor backward ping-pong [B_l][max(width, 2 act)]
  float* ac_phiX[CRL_MAX_LAYERS] = {}; float* ac_phiZ[CRL_MAX_LAYERS] = {};   // critic phi on [s||a']
  float* ac_psiX[CRL_MAX_LAYERS] = {}; float* ac_psiZ[CRL_MAX_LAYERS] = {};   // critic psi on g
  float *ac_phi = nullptr, *ac_psi = nullptr, *ac_dphi = nullptr;            // [B_l][D]
  float* ac_dz[2] = {nullptr, nullptr};    // critic dX chain ping-pong [B_l][max(width, D)]
  float* a_grads = nullptr;                // [dw_splits][n_actor_params]
  float* a_loss = nullptr;                 // [4]: summed rows, summed log pi (all-reduced), loss, mean log pi
  int *a_t = nullptr, *a_skip = nullptr;
  float* a_alpha = nullptr;                // [1] the entropy coefficient of the current actor call
  std::map<ActorKey, std::pair<cudaGraphExec_t, int>> actor_graphs;   // captured actor steps
  std::map<ActorKey, uint64_t> actor_use;  // last replay (LRU eviction beyond kMaxGraphs)
  float* ent_mv = nullptr;                 // [2] Adam moments of log alpha (entropy coefficient)
  int* ent_t = nullptr;                    // its step counter
  bool actor_loss_done = false;            // a crl_actor_loss has produced a mean log pi
};

constexpr int kTcLogitsMinN = 2;         // measured: tensor-core logits win down to N = 256
constexpr int kStatPad = 256;            // padding of per-column arrays read by 1-D bulk copies
constexpr int kChainMinBatch = 8192;     // fused MLP chains from this local batch on (measured)

// Brackets one launch with CUDA events when the context is in profiling mode (events come
// from a pool so the host enqueue stays cheap; see also spin_kernel below).
cudaEvent_t pool_event(crl_ctx* c);
struct Stage {
  crl_ctx* c; cudaStream_t st; cudaEvent_t b = nullptr;
  Stage(crl_ctx* c_, cudaStream_t st_, const std::string& name) : c(c_), st(st_) {
    if (!c->prof_on) return;
    cudaEvent_t a = pool_event(c);
    b = pool_event(c);
    cudaEventRecord(a, st);
    c->prof_pending.push_back({name, a, b});
  }
  ~Stage() { if (b) cudaEventRecord(b, st); }
};

inline crl_status fail(crl_ctx* ctx, crl_status st, const std::string& msg) {
  g_last_error = msg;
  if (ctx) ctx->err = msg;
  return st;
}

#define CU(call)                                                                           \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(ctx, CRL_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
  } while (0)

#define NC(call)                                                                           \
  do {                                                                                     \
    ncclResult_t _r = (call);                                                              \
    if (_r != ncclSuccess)                                                                 \
      return fail(ctx, CRL_ENCCL, std::string(#call) + ": " + ncclGetErrorString(_r));     \
  } while (0)

