// step_bf16.cu — the BF16 tensor-core schedule of crl_critic_step (precision == CRL_BF16):
// bf16 operands everywhere a contraction happens (encoder GEMMs on tcgen05, fed by TMA),
// fp32 accumulation, statistics, loss, gradients and optimiser state.
//
// Per encoder and layer l (W_l stored [in][out], bf16 shadow written by the Adam kernel):
//   fwd  : Z_l = X_l W_l + b_l  -> Z_l (bf16), X_{l+1} = act(Z_l) (bf16)      [output: Y fp32+bf16]
//   dW_l = X_l^T dZ_l  (split-K over the batch, fp32 partial slices), db_l = colsum(dZ_l)
//   dX   : dZ_{l-1} = (dZ_l W_l^T) * act'(Z_{l-1})  (bf16)
// All tensor maps are built once at context creation (buffers are context-owned).
#include "ctx.h"
#include "tc_gradf.h"
#include "tc_merge.cuh"

#include <cstdlib>
#include <vector>

namespace crl {
cudaError_t logits_lse_f32(int, int, const float*, int, const float*, int, float*, cudaStream_t);
cudaError_t logits_grad_f32(int, int, const float*, int, int, const float*, int, const float*,
                            const float*, float, float, float, float, float, float*, cudaStream_t);
cudaError_t launch_loss_partial(const float*, const float*, int, int, int, const float*,
                                const float*, float*, float*, unsigned*, int, float, float, float,
                                float, float*, int*, int*, int*, cudaStream_t);
cudaError_t launch_loss_finalize(const float*, float, float, float, float, float*, int*, int*,
                                 int*, cudaStream_t);
cudaError_t launch_adam(float*, float*, int, float*, float*, size_t, float, float, float, float,
                        float, const int*, const int*, int*, void*, int, cudaStream_t);
cudaError_t launch_adam_ex(float*, float*, int, float*, float*, size_t, float, float, float, float,
                           float, const int*, const int*, int*, void*, int, int, cudaStream_t);
cudaError_t launch_reduce_partials(float*, size_t, int, cudaStream_t);
namespace tc {
bool make_map_bf16(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
bool make_map_f32(CUtensorMap*, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t);
int tc_pick_bn(int M, int N, int num_sms);
cudaError_t tc_forward(int, const CUtensorMap&, const CUtensorMap&, int, int, int, const float*,
                       __nv_bfloat16*, __nv_bfloat16*, int, float*, int, int, float*, int, cudaStream_t);
cudaError_t tc_backward_dx(int, const CUtensorMap&, const CUtensorMap&, int, int, int,
                           const __nv_bfloat16*, __nv_bfloat16*, int, int, cudaStream_t);
cudaError_t tc_backward_dw(int, const CUtensorMap&, const CUtensorMap&, int, int, int, float*, int,
                           size_t, cudaStream_t);
cudaError_t launch_prep_inputs(const float*, const float*, const float*, int, int, int, int,
                               __nv_bfloat16*, int, __nv_bfloat16*, int, int, int*, int*, int, float*, size_t,
                               cudaStream_t);
cudaError_t launch_colsum_bf16(const __nv_bfloat16*, int, int, int, float*, int, size_t, cudaStream_t);
cudaError_t launch_f32_to_bf16(const float*, __nv_bfloat16*, size_t, int, cudaStream_t);
bool tc_logits_maps(CUtensorMap*, CUtensorMap*, const __nv_bfloat16*, int, const __nv_bfloat16*, int, int);
cudaError_t tc_logits_lse(int, int, const CUtensorMap&, const CUtensorMap&, int, int, const float*, const float*,
                          int, float*, float*, float*, float*, int*, float, float, const int*, cudaStream_t);
cudaError_t tc_stats_fused(int, int, const CUtensorMap&, const CUtensorMap&, int, int, const float*, const float*, int,
                           float*, float*, int, float*, float*, float*, float*, int*, int*, float, float, float, float,
                           cudaGraphConditionalHandle, cudaStream_t, float*);
cudaError_t tc_stats_col_finalize(const float*, int, int, float*, float*, int*, int*, float, float, cudaStream_t);
cudaError_t tc_logits_grad(int, int, const CUtensorMap&, const CUtensorMap&, int, int, int, const float*,
                           const float*, const float*, const float*, const float*, float, float, float, float,
                           float, int, float*, float*, const __nv_bfloat16*, const __nv_bfloat16*, float*,
                           __nv_bfloat16*, const int*, cudaStream_t);
cudaError_t launch_rowstat_bf16(const __nv_bfloat16*, int, int, int, float*, int*, int, cudaStream_t);
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st);
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st,
                               const MergeLoss* loss);
cudaError_t launch_grad_merge2(int energy, const GradMergeArgs& g0, const GradMergeArgs& g1, cudaStream_t st,
                               const MergeLoss* loss, int nsides);
}  // namespace tc
}  // namespace crl

using namespace crl;

static crl_status build_encoder_plan(crl_ctx* ctx, const EncoderPlan& P, const __nv_bfloat16* x0, int ld0,
                                     __nv_bfloat16** Xb, __nv_bfloat16** Zb, __nv_bfloat16* dY,
                                     __nv_bfloat16** dzb, float* Yf, __nv_bfloat16* Yb, __nv_bfloat16** LNb,
                                     std::vector<crl_ctx::TcLayer>& out) {
  const int Bl = ctx->cfg.batch_local, Wd = ctx->cfg.width, L = P.n_layers;
  const bool ln = ctx->cfg.layernorm != 0;        // F2: hidden Z -> LN (ln.cu) -> act; LNb[l] = LN(Z_l)
  out.assign(L, crl_ctx::TcLayer{});
  for (int l = 0; l < L; ++l) {
    auto& T = out[l];
    const int in = P.layer[l].in, o = P.layer[l].out;
    const __nv_bfloat16* X = (l == 0) ? x0 : Xb[l];
    const int ldx = (l == 0) ? ld0 : Wd;
    const __nv_bfloat16* W = ctx->wshadow + P.layer[l].w_off;
    T.dz = (l == L - 1) ? dY : dzb[l];
    T.dzprev = (l > 0) ? dzb[l - 1] : nullptr;
    T.bn_fwd = tc::tc_pick_bn(Bl, o, ctx->num_sms);
    T.bn_dw = tc::tc_pick_bn(in, o, ctx->num_sms);
    T.bn_dx = tc::tc_pick_bn(Bl, in, ctx->num_sms);
    bool ok = tc::make_map_bf16(&T.fwdA, X, in, Bl, ldx, 64, 128) &&       // X  K-major
              tc::make_map_bf16(&T.fwdB, W, o, in, o, 64, 64) &&           // W  MN-major (N = out)
              tc::make_map_bf16(&T.dwA, X, in, Bl, ldx, 64, 64) &&         // X  MN-major (M = in)
              tc::make_map_bf16(&T.dwB, T.dz, o, Bl, o, 64, 64);           // dZ MN-major (N = out)
    if (l > 0)
      ok = ok && tc::make_map_bf16(&T.dxA, T.dz, o, Bl, o, 64, 128) &&     // dZ K-major (K = out)
           tc::make_map_bf16(&T.dxB, W, o, in, o, 64, T.bn_dx);            // W  K-major (N = in)
    if (!ok) return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed (driver entry point missing?)");
    // wide layers (width >= 256, 64-aligned): the persistent CTA-pair GEMM; its output row
    // statistic needs the whole representation in one 256-column tile (D <= 256)
    const bool last = l == L - 1;
    T.pg_fwd = tc::tc_pgemm_supported(Bl, o, in) && (!last || o <= 256);
    if (ln && !last && !T.pg_fwd)
      return fail(ctx, CRL_EUNSUPPORTED, "bf16 LayerNorm needs the CTA-pair GEMM for every hidden layer");
    if (T.pg_fwd) {
      T.pgf.a = T.fwdA;
      T.pgf.b = T.fwdB;                                                     // W {out, in} box {64, 64}
      ok = last ? (tc::make_map_f32(&T.pgf.out0, Yf, o, Bl, o, 32, 32) &&
                   tc::make_map_bf16(&T.pgf.out1, Yb, o, Bl, o, 64, 32))
                : (tc::make_map_bf16(&T.pgf.out0, Zb[l], o, Bl, o, 64, 32) &&
                   tc::make_map_bf16(&T.pgf.out1, Xb[l + 1], o, Bl, o, 64, 32));
      if (!ok) return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the CTA-pair GEMM");
    }
    T.pg_dx = l > 0 && tc::tc_pgemm_supported(Bl, in, o);
    if (T.pg_dx) {
      T.pgd.a = T.dxA;                                                      // dZ_l {out, B} box {64, 128}
      ok = tc::make_map_bf16(&T.pgd.b, W, o, in, o, 64, 128) &&            // W K-major {out, in}
           tc::make_map_bf16(&T.pgd.out0, T.dzprev, in, Bl, in, 64, 32) &&
           tc::make_map_bf16(&T.pgd.zin, ln ? LNb[l - 1] : Zb[l - 1], in, Bl, in, 64, 32);   // act' at Y (LN) / Z
      if (!ok) return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the CTA-pair GEMM");
    }
    if (ln && l > 0 && !T.pg_dx)
      return fail(ctx, CRL_EUNSUPPORTED, "bf16 LayerNorm needs the CTA-pair GEMM for every dX product");
  }
  return CRL_OK;
}

crl_status bf16_prepare(crl_ctx* ctx) {
  const crl_config& k = ctx->cfg;
  crl_status st = build_encoder_plan(ctx, ctx->phi_plan, ctx->x0_phi, ctx->ld0_phi, ctx->phiXb, ctx->phiZb,
                                     ctx->dphib, ctx->dzb_phi, ctx->phi_out, ctx->phi_outb, ctx->phiYb, ctx->tc_phi);
  if (st != CRL_OK) return st;
  st = build_encoder_plan(ctx, ctx->psi_plan, ctx->x0_psi, ctx->ld0_psi, ctx->psiXb, ctx->psiZb, ctx->dpsib,
                          ctx->dzb_psi, ctx->psi_out, ctx->psi_outb, ctx->psiYb, ctx->tc_psi);
  if (st != CRL_OK) return st;
  // grouped weight / bias gradients: X_l and dZ_l of every layer of both encoders
  // wide encoders (configs[4]: width 1024): every dW / db on CTA pairs, 256 x 256 tiles
  ctx->use_pdw = k.width >= 512 && tc::pdw_supported(k.batch_local, ctx->dw_splits);
  if (ctx->use_pdw) {
    tc::pdw_init(ctx->pdw, k.batch_local, ctx->dw_splits, ctx->sizes.n_params);
    ctx->pdw_split = !ctx->dist && !std::getenv("CRL_NO_PDW_SPLIT");
    if (ctx->pdw_split) tc::pdw_init(ctx->pdw_psi, k.batch_local, ctx->dw_splits, ctx->sizes.n_params);
    const EncoderPlan* plans[2] = {&ctx->phi_plan, &ctx->psi_plan};
    std::vector<crl_ctx::TcLayer>* tcs[2] = {&ctx->tc_phi, &ctx->tc_psi};
    __nv_bfloat16** Xb[2] = {ctx->phiXb, ctx->psiXb};
    const __nv_bfloat16* x0[2] = {ctx->x0_phi, ctx->x0_psi};
    const int ld0[2] = {ctx->ld0_phi, ctx->ld0_psi};
    // problem order = work-item order: the pairs take items round-robin, so the first layers
    // (K = in <= 37: their X tiles are mostly TMA zero-fill, about half the operand traffic of
    // a full item) go LAST and fill the final partial round (makespan 3.5 instead of 4 items
    // at netscale: 208 full + 16 half items on 74 pairs)
    const int L = plans[0]->n_layers;
    const bool natural = std::getenv("CRL_PDW_NATURAL_ORDER") != nullptr;   // measurement knob
    for (int pass = 0; pass < (natural ? 1 : 2) && ctx->use_pdw; ++pass)
    for (int e = 0; e < 2 && ctx->use_pdw; ++e)
      for (int l = natural ? 0 : (pass == 0 ? 1 : 0); l < (natural || pass == 0 ? L : 1); ++l) {
        const LayerPlan& Lp = plans[e]->layer[l];
        if (!tc::pdw_add_problem(e == 1 && ctx->pdw_split ? ctx->pdw_psi : ctx->pdw, l == 0 ? x0[e] : Xb[e][l],
                                 l == 0 ? ld0[e] : k.width, (*tcs[e])[l].dz, Lp.in, Lp.out, ctx->grads + Lp.w_off,
                                 ctx->grads + Lp.b_off)) {
          ctx->use_pdw = false;                 // (alignment / table size): the grouped kernel
          break;
        }
      }
  }
  ctx->use_dwg = !ctx->use_pdw && !std::getenv("CRL_NO_DWG");
  if (ctx->use_dwg) {
    tc::dwg_init(ctx->dwg, k.batch_local, ctx->dw_splits, ctx->sizes.n_params);
    const EncoderPlan* plans[2] = {&ctx->phi_plan, &ctx->psi_plan};
    std::vector<crl_ctx::TcLayer>* tcs[2] = {&ctx->tc_phi, &ctx->tc_psi};
    __nv_bfloat16** Xb[2] = {ctx->phiXb, ctx->psiXb};
    const __nv_bfloat16* x0[2] = {ctx->x0_phi, ctx->x0_psi};
    const int ld0[2] = {ctx->ld0_phi, ctx->ld0_psi};
    for (int e = 0; e < 2; ++e)
      for (int l = 0; l < plans[e]->n_layers; ++l) {
        const LayerPlan& Lp = plans[e]->layer[l];
        if (!tc::dwg_add_problem(ctx->dwg, l == 0 ? x0[e] : Xb[e][l], l == 0 ? ld0[e] : k.width, (*tcs[e])[l].dz,
                                 Lp.in, Lp.out, ctx->grads + Lp.w_off, ctx->grads + Lp.b_off))
          return fail(ctx, CRL_ECUDA, "grouped weight-gradient setup failed (tensor maps)");
      }
  }
  if (ctx->tc_logits) {
    ctx->lg_splits = std::min(ctx->lg_splits, tc::tc_logits_splits(k.batch_local, ctx->N, k.repr_dim,
                                                                   ctx->num_sms));
    if (!tc::tc_logits_maps(&ctx->lg_row_A, &ctx->lg_row_B, ctx->phi_outb, k.batch_local, ctx->psi_outb_g,
                            ctx->N, k.repr_dim) ||
        !tc::tc_logits_maps(&ctx->lg_col_A, &ctx->lg_col_B, ctx->psi_outb, k.batch_local, ctx->phi_outb_g,
                            ctx->N, k.repr_dim))
      return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the logits operands");
    if (ctx->use_grad2) {
      if (!tc::make_map_bf16(&ctx->g2_B0, ctx->psi_outb_g, k.repr_dim, ctx->N, k.repr_dim, 64, 128) ||
          !tc::make_map_bf16(&ctx->g2_B1, ctx->phi_outb_g, k.repr_dim, ctx->N, k.repr_dim, 64, 128))
        return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the gradient operands");
      const int RB = (k.batch_local + 127) / 128;
      std::vector<unsigned char> fl(2 * RB);
      if (ctx->g2_pair) {
        if (!tc::make_map_bf16(&ctx->g2_S0, ctx->psi_outb_g, k.repr_dim, ctx->N, k.repr_dim, 64, 64) ||
            !tc::make_map_bf16(&ctx->g2_S1, ctx->phi_outb_g, k.repr_dim, ctx->N, k.repr_dim, 64, 64) ||
            !tc::make_map_bf16(&ctx->g2_A0, ctx->phi_outb, k.repr_dim, k.batch_local, k.repr_dim, 64, 128) ||
            !tc::make_map_bf16(&ctx->g2_A1, ctx->psi_outb, k.repr_dim, k.batch_local, k.repr_dim, 64, 128))
          return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the gradient operands");
        const int pieces = tc::tc_grad2p_split_flags(k.batch_local, ctx->N, ctx->g2_grid, fl.data(),
                                                     ctx->g2_wsym ? 1 : 2);
        if (pieces > (ctx->g2_wsym ? 3 : 2))
          return fail(ctx, CRL_EUNSUPPORTED, "gradient pass: a row block cut into more pieces than partial slots");
        if (ctx->g2_wsym) {
          // W (bf16 [B_l][N]) and dPsi slots 0 / 1 = the two K halves of W^T Phi, column sums beside
          const int Bl = k.batch_local, D = k.repr_dim, ldw = (ctx->N + 63) / 64 * 64;
          // (Phi^T W on 256 x 512 items: the Phi K block is shared by 512 columns of W; 2 K slices
          // give 64 items, one wave of pairs; the result is stored transposed, i.e. [N][256])
          tc::pdw_init(ctx->pdw_g, Bl, 2, 0);
          if (!tc::make_map_bf16(&ctx->g2_Wmap, ctx->g2_W, ctx->N, Bl, ldw, 64, 128) ||
              !tc::pdw_add_gemm_t(ctx->pdw_g, ctx->phi_outb, D, ctx->g2_W, ldw, D, ctx->N,
                                  ctx->g2_part_da + (size_t)3 * Bl * D, (long long)Bl * D, ctx->g2_cs, ctx->N))
            return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the stored gradient weights");
        }
      } else {
        tc::tc_grad2_split_flags(k.batch_local, ctx->N, ctx->g2_grid, fl.data());
      }
      CU(cudaMemcpy(ctx->g2_flags, fl.data(), fl.size(), cudaMemcpyHostToDevice));
    }
    if (ctx->use_stats && (!tc::make_map_bf16(&ctx->st_A, ctx->phi_outb, k.repr_dim, k.batch_local, k.repr_dim, 64, 128) ||
                           !tc::make_map_bf16(&ctx->st_B, ctx->psi_outb_g, k.repr_dim, ctx->N, k.repr_dim, 64, 128)))
      return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the statistics operands");
    if (ctx->use_gradf && !tc::tc_gradf_map(&ctx->gf_map, ctx->gf_acc, ctx->N))
      return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the column-gradient accumulator");
  }
  // fused MLP chains (activations resident in SMEM/TMEM across layers) when the shapes fit
  // (measured on B200: the chain wins from B_l = 8192 on; below it the per-layer GEMMs, which
  // spread each layer over more SMs, are as fast or faster.  CRL_CHAIN / CRL_NO_CHAIN force it.)
  // The cluster chains below (4 CTAs per 128 rows and encoder) win while they fit in one wave;
  // once 8 ceil(B_l / 128) CTAs exceed the SM count the per-row-block chain is faster (measured:
  // B_l = 2048 cchain 114 us/step vs chain 135; B_l = 4096 cchain 175 vs chain 165).
  const bool cchain_shapes = tc::tc_cchain_supported(k.obs_dim + k.act_dim, k.width, k.repr_dim, k.depth) &&
                             tc::tc_cchain_supported(k.goal_dim, k.width, k.repr_dim, k.depth);
  const bool cchain_one_wave = 8 * ((k.batch_local + 127) / 128) <= ctx->num_sms;
  const bool chain_wanted = std::getenv("CRL_CHAIN") ? true
                            : std::getenv("CRL_NO_CHAIN") ? false
                            : (k.batch_local >= kChainMinBatch || (cchain_shapes && !cchain_one_wave &&
                                                                   !std::getenv("CRL_CCHAIN")));
  ctx->use_chain = ctx->tc_logits && chain_wanted && k.depth >= 1 && !k.layernorm &&
                   tc::tc_chain_supported(k.obs_dim + k.act_dim, k.width, k.repr_dim, k.depth) &&
                   tc::tc_chain_supported(k.goal_dim, k.width, k.repr_dim, k.depth);
  if (ctx->use_chain) {
    const int row_off = k.rank * k.batch_local;
    const EncoderPlan* plans[2] = {&ctx->phi_plan, &ctx->psi_plan};
    std::vector<crl_ctx::TcLayer>* tcs[2] = {&ctx->tc_phi, &ctx->tc_psi};
    __nv_bfloat16** Xb[2] = {ctx->phiXb, ctx->psiXb};
    __nv_bfloat16** Zb[2] = {ctx->phiZb, ctx->psiZb};
    __nv_bfloat16** dzb[2] = {ctx->dzb_phi, ctx->dzb_psi};
    __nv_bfloat16* Yb[2] = {ctx->phi_outb, ctx->psi_outb};
    float* Yf[2] = {ctx->phi_out, ctx->psi_out};
    float* stat[2] = {ctx->stat_phi + row_off, ctx->stat_psi + row_off};
    tc::ChainParams& F = ctx->chain_fwd_p;
    tc::ChainParams& Bw = ctx->chain_bwd_p;
    F.M = Bw.M = k.batch_local;
    F.act = Bw.act = k.activation;
    F.energy = Bw.energy = k.energy;
    F.fac_ok = ctx->fac_ok;
    F.fac_init = std::getenv("CRL_FORCE_EXACT_Q") ? 0 : 1;
    F.dbg = Bw.dbg = std::getenv("CRL_CHAIN_DBG") ? std::atoi(std::getenv("CRL_CHAIN_DBG")) : 0;
    Bw.fac_ok = nullptr;
    for (int e = 0; e < 2; ++e) {
      const EncoderPlan& P = *plans[e];
      const int L = P.n_layers;
      auto& T = *tcs[e];
      tc::ChainEnc& fe = F.enc[e];
      tc::ChainEnc& be = Bw.enc[e];
      fe.L = L;
      fe.out_stat = stat[e];
      ctx->chain_fwd[e].a0 = T[0].fwdA;
      for (int l = 0; l < L; ++l) {
        const LayerPlan& Lp = P.layer[l];
        tc::ChainLayer& cl = fe.layer[l];
        cl.K = Lp.in; cl.N = Lp.out;
        cl.bias = ctx->mem.params + Lp.b_off;
        cl.out_act = (l < L - 1) ? Xb[e][l + 1] : Yb[e];
        cl.out_z = (l < L - 1) ? Zb[e][l] : nullptr;
        cl.out_f = (l == L - 1) ? Yf[e] : nullptr;
        ctx->chain_fwd[e].w[l] = T[l].fwdB;
        // TMA-store targets: whole 128 x 64 chunks straight from the kernel's SW128 SMEM buffers
        bool ok = tc::make_map_bf16(&ctx->chain_fwd[e].st_out[l], cl.out_act, Lp.out, k.batch_local, Lp.out, 64,
                                    128);
        if (l < L - 1)
          ok = ok && tc::make_map_bf16(&ctx->chain_fwd[e].st_z[l], cl.out_z, Lp.out, k.batch_local, Lp.out, 64,
                                       128);
        if (!ok) return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the chain outputs");
      }
      be.L = L - 1;
      be.out_stat = nullptr;
      ctx->chain_bwd[e].a0 = T[L - 1].dxA;                 // dY, K-major box {64, 128}
      for (int s2 = 0; s2 < L - 1; ++s2) {
        const int l = L - 1 - s2;
        const LayerPlan& Lp = P.layer[l];
        tc::ChainLayer& cl = be.layer[s2];
        cl.K = Lp.out; cl.N = Lp.in;
        cl.out_act = dzb[e][l - 1];
        cl.zprev = Zb[e][l - 1];
        if (!tc::make_map_bf16(&ctx->chain_bwd[e].w[s2], ctx->wshadow + Lp.w_off, Lp.out, Lp.in, Lp.out, 64,
                               Lp.in) ||
            !tc::make_map_bf16(&ctx->chain_bwd[e].st_out[s2], cl.out_act, Lp.in, k.batch_local, Lp.in, 64, 128))
          return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the chain weights");
      }
    }
  }
  // cluster-split chains for the small batches the per-row-block chain does not cover
  ctx->use_cchain = !ctx->use_chain && ctx->tc_logits && !std::getenv("CRL_NO_CCHAIN") && !k.layernorm &&
                    (std::getenv("CRL_CCHAIN") || k.batch_local < kChainMinBatch) && cchain_shapes;
  if (ctx->use_cchain) {
    const int Bl = k.batch_local, row_off = k.rank * Bl;
    const EncoderPlan* plans[2] = {&ctx->phi_plan, &ctx->psi_plan};
    std::vector<crl_ctx::TcLayer>* tcs[2] = {&ctx->tc_phi, &ctx->tc_psi};
    __nv_bfloat16** Xb[2] = {ctx->phiXb, ctx->psiXb};
    __nv_bfloat16** Zb[2] = {ctx->phiZb, ctx->psiZb};
    __nv_bfloat16** dzb[2] = {ctx->dzb_phi, ctx->dzb_psi};
    __nv_bfloat16* Yb[2] = {ctx->phi_outb, ctx->psi_outb};
    float* Yf[2] = {ctx->phi_out, ctx->psi_out};
    float* stat[2] = {ctx->stat_phi + row_off, ctx->stat_psi + row_off};
    tc::CChainParams& F = ctx->cchain_fwd_p;
    tc::CChainParams& Bw = ctx->cchain_bwd_p;
    F = tc::CChainParams{};
    Bw = tc::CChainParams{};
    F.M = Bw.M = Bl;
    F.act = Bw.act = k.activation;
    F.energy = Bw.energy = k.energy;
    F.store_ok = Bw.store_ok = std::getenv("CRL_CCHAIN_NOSTORE") ? 0 : 1;
    F.trace = Bw.trace = std::getenv("CRL_CCHAIN_TRACE") ? 1 : 0;
    for (int e = 0; e < 2; ++e) {
      const EncoderPlan& P = *plans[e];
      const int L = P.n_layers;
      auto& T = *tcs[e];
      tc::CChainEnc& fe = F.enc[e];
      tc::CChainEnc& be = Bw.enc[e];
      fe.L = L;
      fe.out_stat = stat[e];
      ctx->cchain_fwd[e].a0 = T[0].fwdA;
      bool ok = true;
      for (int l = 0; l < L; ++l) {
        const LayerPlan& Lp = P.layer[l];
        tc::CChainLayer& cl = fe.layer[l];
        cl.K = Lp.in; cl.N = Lp.out;
        cl.bias = ctx->mem.params + Lp.b_off;
        cl.out_z = (l < L - 1) ? Zb[e][l] : nullptr;
        cl.out_act = (l == L - 1) ? Yb[e] : nullptr;
        cl.out_f = (l == L - 1) ? Yf[e] : nullptr;
        ctx->cchain_fwd[e].w[l] = T[l].fwdB;                      // W_l {out, in}, box {64, 64}
        if (l < L - 1) ok = ok && tc::make_map_bf16(&ctx->cchain_fwd[e].st[l], Xb[e][l + 1], Lp.out, Bl, Lp.out, 64, 128);
      }
      be.L = L - 1;
      be.out_stat = nullptr;
      ctx->cchain_bwd[e].a0 = T[L - 1].dxA;                       // dY, box {64, 128}
      for (int s2 = 0; s2 < L - 1; ++s2) {
        const int l = L - 1 - s2;
        const LayerPlan& Lp = P.layer[l];
        tc::CChainLayer& cl = be.layer[s2];
        cl.K = Lp.out; cl.N = Lp.in;
        cl.zprev = Zb[e][l - 1];
        ctx->cchain_bwd[e].w[s2] = T[l].fwdB;                     // the same bytes, read K-major
        ok = ok && tc::make_map_bf16(&ctx->cchain_bwd[e].st[s2], dzb[e][l - 1], Lp.in, Bl, Lp.in, 64, 128);
      }
      if (!ok) return fail(ctx, CRL_ECUDA, "cuTensorMapEncodeTiled failed for the cluster chains");
    }
  }
  // initial bf16 shadow of the caller's parameters; zero the padded input rows
  CU(tc::launch_f32_to_bf16(ctx->mem.params, ctx->wshadow, ctx->sizes.n_params, ctx->num_sms, 0));
  CU(cudaMemset(ctx->x0_phi, 0, (size_t)k.batch_local * ctx->ld0_phi * 2));
  CU(cudaMemset(ctx->x0_psi, 0, (size_t)k.batch_local * ctx->ld0_psi * 2));
  CU(cudaDeviceSynchronize());
  return CRL_OK;
}

static crl_status enc_forward_bf16(crl_ctx* ctx, const char* tag, const EncoderPlan& P,
                                   std::vector<crl_ctx::TcLayer>& T, __nv_bfloat16** Xb, __nv_bfloat16** Zb,
                                   float* yf, __nv_bfloat16* yb, float* ystat, cudaStream_t st, int* nl) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, L = P.n_layers;
  for (int l = 0; l < L; ++l) {
    const LayerPlan& Lp = P.layer[l];
    const bool last = l == L - 1;
    Stage sg(ctx, st, std::string(tag) + "_fwd_l" + std::to_string(l));
    if (T[l].pg_fwd) {
      tc::PgemmArgs pa{Bl, Lp.out, Lp.in, ctx->mem.params + Lp.b_off, k.activation, last ? ystat : nullptr,
                       k.energy};
      pa.lin = (k.layernorm && !last) ? 1 : 0;          // LN: Z only, then the LayerNorm kernel
      CU(tc::tc_pgemm(last ? tc::PG_FWD_OUT : tc::PG_FWD_HIDDEN, T[l].pgf, pa, ctx->num_sms, st));
      if (pa.lin) {
        const bool phi = Xb == ctx->phiXb;
        CU(launch_ln_fwd_bf16(Bl, Lp.out, Zb[l], ctx->mem.params + Lp.g_off, ctx->mem.params + Lp.be_off,
                              k.activation, phi ? ctx->phiYb[l] : ctx->psiYb[l], Xb[l + 1],
                              phi ? ctx->phiMu[l] : ctx->psiMu[l], phi ? ctx->phiRs[l] : ctx->psiRs[l], st));
        ++*nl;
      }
    } else {
      CU(tc::tc_forward(T[l].bn_fwd, T[l].fwdA, T[l].fwdB, Bl, Lp.in, Lp.out, ctx->mem.params + Lp.b_off,
                        last ? nullptr : Zb[l], last ? yb : Xb[l + 1], Lp.out, last ? yf : nullptr, Lp.out,
                        k.activation, last ? ystat : nullptr, k.energy, st));
    }
    ++*nl;
  }
  return CRL_OK;
}

// The phi and psi encoders have the same depth and width: with CTA-pair GEMMs on every layer,
// layer l of both runs as ONE persistent launch (tc_pgemm2: one wave quantisation for 2 x 256
// tiles instead of two, half the launches) instead of two kernels on two streams.
static bool pg_pair_layers(const crl_ctx* ctx, bool dx) {
  if (std::getenv("CRL_NO_PG_MERGE")) return false;
  const EncoderPlan &A = ctx->phi_plan, &B = ctx->psi_plan;
  if (A.n_layers != B.n_layers) return false;
  for (int l = dx ? 1 : 0; l < A.n_layers; ++l) {
    const bool a = dx ? ctx->tc_phi[l].pg_dx : ctx->tc_phi[l].pg_fwd;
    const bool b = dx ? ctx->tc_psi[l].pg_dx : ctx->tc_psi[l].pg_fwd;
    if (!a || !b || A.layer[l].out != B.layer[l].out) return false;
  }
  return true;
}

static crl_status enc_forward_pair_bf16(crl_ctx* ctx, float* stat_phi, float* stat_psi, cudaStream_t st, int* nl) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, L = ctx->phi_plan.n_layers;
  for (int l = 0; l < L; ++l) {
    const bool last = l == L - 1;
    Stage sg(ctx, st, "enc_fwd_l" + std::to_string(l));
    tc::PgemmArgs pa[2];
    const EncoderPlan* P[2] = {&ctx->phi_plan, &ctx->psi_plan};
    float* stat[2] = {stat_phi, stat_psi};
    for (int e = 0; e < 2; ++e) {
      const LayerPlan& Lp = P[e]->layer[l];
      pa[e] = tc::PgemmArgs{Bl, Lp.out, Lp.in, ctx->mem.params + Lp.b_off, k.activation, last ? stat[e] : nullptr,
                            k.energy};
      pa[e].lin = (k.layernorm && !last) ? 1 : 0;
    }
    CU(tc::tc_pgemm2(last ? tc::PG_FWD_OUT : tc::PG_FWD_HIDDEN, ctx->tc_phi[l].pgf, pa[0], ctx->tc_psi[l].pgf,
                     pa[1], ctx->num_sms, st));
    ++*nl;
    if (pa[0].lin) {
      for (int e = 0; e < 2; ++e) {
        const LayerPlan& Lp = P[e]->layer[l];
        const bool phi = e == 0;
        CU(launch_ln_fwd_bf16(Bl, Lp.out, phi ? ctx->phiZb[l] : ctx->psiZb[l], ctx->mem.params + Lp.g_off,
                              ctx->mem.params + Lp.be_off, k.activation, phi ? ctx->phiYb[l] : ctx->psiYb[l],
                              phi ? ctx->phiXb[l + 1] : ctx->psiXb[l + 1], phi ? ctx->phiMu[l] : ctx->psiMu[l],
                              phi ? ctx->phiRs[l] : ctx->psiRs[l], st));
        ++*nl;
      }
    }
  }
  return CRL_OK;
}

static crl_status enc_backward_pair_bf16(crl_ctx* ctx, cudaStream_t st, int* nl) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, L = ctx->phi_plan.n_layers;
  for (int l = L - 1; l >= 1; --l) {
    Stage sg(ctx, st, "enc_bwd_dx_l" + std::to_string(l));
    tc::PgemmArgs pa[2];
    const EncoderPlan* P[2] = {&ctx->phi_plan, &ctx->psi_plan};
    for (int e = 0; e < 2; ++e) {
      const LayerPlan& Lp = P[e]->layer[l];
      pa[e] = tc::PgemmArgs{Bl, Lp.in, Lp.out, nullptr, k.activation, nullptr, k.energy};
    }
    CU(tc::tc_pgemm2(tc::PG_DX, ctx->tc_phi[l].pgd, pa[0], ctx->tc_psi[l].pgd, pa[1], ctx->num_sms, st));
    ++*nl;
    if (k.layernorm) {                                  // dY_{l-1} (act' at Y) -> dZ_{l-1}, dgamma, dbeta
      for (int e = 0; e < 2; ++e) {
        const bool phi = e == 0;
        const LayerPlan& Lq = P[e]->layer[l - 1];
        std::vector<crl_ctx::TcLayer>& T = phi ? ctx->tc_phi : ctx->tc_psi;
        CU(launch_ln_bwd_bf16(Bl, Lq.out, T[l].dzprev, phi ? ctx->phiZb[l - 1] : ctx->psiZb[l - 1],
                              phi ? ctx->phiMu[l - 1] : ctx->psiMu[l - 1], phi ? ctx->phiRs[l - 1] : ctx->psiRs[l - 1],
                              ctx->mem.params + Lq.g_off, phi ? ctx->ln_part_phi : ctx->ln_part_psi, ctx->ln_nblk,
                              ctx->grads + Lq.g_off, ctx->grads + Lq.be_off, ctx->dw_splits, ctx->sizes.n_params, st));
        *nl += 2;
      }
    }
  }
  return CRL_OK;
}

static crl_status enc_backward_bf16(crl_ctx* ctx, const char* tag, const EncoderPlan& P,
                                    std::vector<crl_ctx::TcLayer>& T, __nv_bfloat16** Zb, cudaStream_t st,
                                    cudaStream_t side, int* nl) {
  const crl_config& k = ctx->cfg;
  const int Bl = k.batch_local, L = P.n_layers;
  for (int l = L - 1; l >= 0; --l) {
    const LayerPlan& Lp = P.layer[l];
    // dW_l and db_l only feed Adam: they run on a side stream, off the dX critical path
    // (or all at once in the grouped kernel after both dX chains: ctx->use_dwg)
    if (side != st && !ctx->use_dwg && !ctx->use_pdw) {
      cudaEventRecord(ctx->ev_side, st);
      cudaStreamWaitEvent(side, ctx->ev_side, 0);
    }
    if (!ctx->use_dwg && !ctx->use_pdw) {
      Stage sg(ctx, side, std::string(tag) + "_bwd_dw_l" + std::to_string(l));
      CU(tc::tc_backward_dw(T[l].bn_dw, T[l].dwA, T[l].dwB, Bl, Lp.in, Lp.out, ctx->grads + Lp.w_off,
                            ctx->dw_splits, ctx->sizes.n_params, side));
      ++*nl;
    }
    if (!ctx->use_dwg && !ctx->use_pdw) {
      Stage sg(ctx, side, std::string(tag) + "_bwd_db_l" + std::to_string(l));
      CU(tc::launch_colsum_bf16(T[l].dz, Bl, Lp.out, Lp.out, ctx->grads + Lp.b_off, ctx->dw_splits,
                                ctx->sizes.n_params, side));
      ++*nl;
    }
    if (l > 0) {
      Stage sg(ctx, st, std::string(tag) + "_bwd_dx_l" + std::to_string(l));
      if (T[l].pg_dx) {
        const tc::PgemmArgs pa{Bl, Lp.in, Lp.out, nullptr, k.activation, nullptr, k.energy};
        CU(tc::tc_pgemm(tc::PG_DX, T[l].pgd, pa, ctx->num_sms, st));
        if (k.layernorm) {                              // dY_{l-1} (act' at Y) -> dZ_{l-1}, dgamma, dbeta
          const LayerPlan& Lq = P.layer[l - 1];
          const bool phi = Zb == ctx->phiZb;
          CU(launch_ln_bwd_bf16(Bl, Lq.out, T[l].dzprev, Zb[l - 1], phi ? ctx->phiMu[l - 1] : ctx->psiMu[l - 1],
                                phi ? ctx->phiRs[l - 1] : ctx->psiRs[l - 1], ctx->mem.params + Lq.g_off,
                                phi ? ctx->ln_part_phi : ctx->ln_part_psi, ctx->ln_nblk, ctx->grads + Lq.g_off,
                                ctx->grads + Lq.be_off, ctx->dw_splits, ctx->sizes.n_params, st));
          *nl += 2;
        }
      } else {
        CU(tc::tc_backward_dx(T[l].bn_dx, T[l].dxA, T[l].dxB, Bl, Lp.in, Lp.out, Zb[l - 1], T[l].dzprev, Lp.in,
                              k.activation, st));
      }
      ++*nl;
    }
  }
  return CRL_OK;
}

// dW_l and db_l of every layer (after the fused dX chain wrote all dZ_l), on one stream
static crl_status enc_weight_grads_bf16(crl_ctx* ctx, const char* tag, const EncoderPlan& P,
                                        std::vector<crl_ctx::TcLayer>& T, cudaStream_t st, int* nl) {
  const int Bl = ctx->cfg.batch_local;
  for (int l = P.n_layers - 1; l >= 0; --l) {
    const LayerPlan& Lp = P.layer[l];
    {
      Stage sg(ctx, st, std::string(tag) + "_bwd_dw_l" + std::to_string(l));
      CU(tc::tc_backward_dw(T[l].bn_dw, T[l].dwA, T[l].dwB, Bl, Lp.in, Lp.out, ctx->grads + Lp.w_off,
                            ctx->dw_splits, ctx->sizes.n_params, st));
      ++*nl;
    }
    {
      Stage sg(ctx, st, std::string(tag) + "_bwd_db_l" + std::to_string(l));
      CU(tc::launch_colsum_bf16(T[l].dz, Bl, Lp.out, Lp.out, ctx->grads + Lp.b_off, ctx->dw_splits,
                                ctx->sizes.n_params, st));
      ++*nl;
    }
  }
  return CRL_OK;
}

static void fork2(crl_ctx* ctx, cudaStream_t s0, cudaStream_t s1) {
  if (s0 == s1) return;
  cudaEventRecord(ctx->ev_fork, s0);
  cudaStreamWaitEvent(s1, ctx->ev_fork, 0);
}
static void join2(crl_ctx* ctx, cudaStream_t s0, cudaStream_t s1) {
  if (s0 == s1) return;
  cudaEventRecord(ctx->ev_join, s1);
  cudaStreamWaitEvent(s0, ctx->ev_join, 0);
}

crl_status enqueue_critic_bf16(crl_ctx* ctx, const float* s, const float* a, const float* g, float* loss_out,
                               float* grads_out, cudaStream_t st, cudaStream_t st2) {
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
  const int row_off = k.rank * Bl;
  // the per-row statistic of Y comes out of the last forward layer's epilogue when that
  // layer's output row fits one CTA (else a separate row-statistic launch)
  auto stat_fits = [&](const crl_ctx::TcLayer& T) { return T.pg_fwd ? D <= 256 : D <= T.bn_fwd; };
  const bool stat_in_fwd = ctx->tc_logits && !ctx->use_chain && stat_fits(ctx->tc_phi.back()) &&
                           stat_fits(ctx->tc_psi.back());
  {
    Stage sg(ctx, st, "prep_inputs");
    // also re-arms the step's device flags (fused-stats fallback gate, fast-factor flag)
    CU(tc::launch_prep_inputs(s, a, g, Bl, k.obs_dim, k.act_dim, k.goal_dim, ctx->x0_phi, ctx->ld0_phi,
                              ctx->x0_psi, ctx->ld0_psi, ctx->num_sms, ctx->use_stats ? ctx->st_bad : nullptr,
                              ctx->tc_logits ? ctx->fac_ok : nullptr, std::getenv("CRL_FORCE_EXACT_Q") ? 0 : 1,
                              ctx->use_gradf ? ctx->gf_acc : nullptr, ctx->use_gradf ? ctx->gf_acc_bytes / 4 : 0,
                              st));
    ++nl;
  }
  if (ctx->use_chain) {
    // both encoders, every layer, one launch; also emits the row statistics of Y
    Stage sg(ctx, st, "mlp_fwd_chain");
    CU(tc::tc_chain_forward(ctx->chain_fwd[0], ctx->chain_fwd[1], ctx->chain_fwd_p, st));
    ++nl;
  } else if (ctx->use_cchain) {
    // both encoders, every layer, one launch of 4-CTA clusters; also the row statistics of Y
    Stage sg(ctx, st, "mlp_fwd_cchain");
    CU(tc::tc_cchain_forward(ctx->cchain_fwd[0], ctx->cchain_fwd[1], ctx->cchain_fwd_p, st));
    ++nl;
  } else if (pg_pair_layers(ctx, false)) {
    rs = enc_forward_pair_bf16(ctx, stat_in_fwd ? ctx->stat_phi + row_off : nullptr,
                               stat_in_fwd ? ctx->stat_psi + row_off : nullptr, st, &nl);
    if (rs != CRL_OK) return rs;
  } else {
    fork2(ctx, st, st2);
    rs = enc_forward_bf16(ctx, "psi", ctx->psi_plan, ctx->tc_psi, ctx->psiXb, ctx->psiZb, ctx->psi_out,
                          ctx->psi_outb, stat_in_fwd ? ctx->stat_psi + row_off : nullptr, st2, &nl);
    if (rs != CRL_OK) return rs;
    rs = enc_forward_bf16(ctx, "phi", ctx->phi_plan, ctx->tc_phi, ctx->phiXb, ctx->phiZb, ctx->phi_out,
                          ctx->phi_outb, stat_in_fwd ? ctx->stat_phi + row_off : nullptr, st, &nl);
    if (rs != CRL_OK) return rs;
    join2(ctx, st, st2);
  }
  const int S = ctx->lg_splits;
  if (ctx->tc_logits) {
    // per-row |x|^2 (L2) / 1/|x| (cos) of the bf16-rounded representations
    if (!ctx->use_chain && !ctx->use_cchain && !stat_in_fwd) { Stage sg(ctx, st, "rowstat");
      const int fac_init = std::getenv("CRL_FORCE_EXACT_Q") ? 0 : 1;
      CU(tc::launch_rowstat_bf16(ctx->phi_outb, Bl, D, k.energy, ctx->stat_phi + row_off, ctx->fac_ok, fac_init,
                                 st));
      CU(tc::launch_rowstat_bf16(ctx->psi_outb, Bl, D, k.energy, ctx->stat_psi + row_off, nullptr, 1, st));
      nl += 2; }
    if (ctx->dist) {   // global negatives: gather the bf16 representations and their statistics
      NC(ncclGroupStart());
      NC(ncclAllGather(ctx->phi_outb, ctx->phi_outb_g, (size_t)Bl * D, ncclBfloat16, ctx->comm, st));
      NC(ncclAllGather(ctx->psi_outb, ctx->psi_outb_g, (size_t)Bl * D, ncclBfloat16, ctx->comm, st));
      NC(ncclAllGather(ctx->stat_phi + row_off, ctx->stat_phi, (size_t)Bl, ncclFloat32, ctx->comm, st));
      NC(ncclAllGather(ctx->stat_psi + row_off, ctx->stat_psi, (size_t)Bl, ncclFloat32, ctx->comm, st));
      NC(ncclGroupEnd());
    }
    const int* gate = nullptr;
    cudaGraphConditionalHandle cond = 0;
    // the two-call online-max statistics, both sides in one launch (merged in-kernel):
    // row side A = Phi (lse_row / fac_row, penalty coefficient), column side A = Psi
    const tc::LseSide row_side{&ctx->lg_row_A, &ctx->lg_row_B, ctx->stat_phi + row_off, ctx->stat_psi,
                               ctx->lg_part_m, ctx->lg_part_s, ctx->lse_row, ctx->fac_row, invN * c_f,
                               2.f * invN * k.beta_lse};
    const tc::LseSide col_side{&ctx->lg_col_A, &ctx->lg_col_B, ctx->stat_psi + row_off, ctx->stat_phi,
                               ctx->lg_part_m + (size_t)S * Bl, ctx->lg_part_s + (size_t)S * Bl, ctx->lse_col,
                               ctx->fac_col, invN * c_b, 0.f};
    if (ctx->use_stats) {
      // one pass: row AND column sums of e^l (no running max: L2 / cos logits are bounded
      // above); the exact online-max pass below then runs only if a sum under/overflowed:
      // by default as early-exit gated kernels.  CRL_COND_NODE=1 instead captures it as the
      // body of a conditional (IF) graph node set by the merge kernel -- measured slower on
      // B200 (ant: 99 -> 107 us/step: the node breaks the programmatic-launch chain).
      if (st != st2 && std::getenv("CRL_COND_NODE")) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaGraph_t cg = nullptr;
        CU(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, nullptr, nullptr));
        if (cs == cudaStreamCaptureStatusActive && cg != nullptr)
          CU(cudaGraphConditionalHandleCreate(&cond, cg, 0, cudaGraphCondAssignDefault));
      }
      Stage sg(ctx, st, "lse_fused");
      CU(tc::tc_stats_fused(D, k.energy, ctx->st_A, ctx->st_B, Bl, N, ctx->stat_phi + row_off, ctx->stat_psi,
                            ctx->st_splits, ctx->st_part_rs, ctx->st_colpart, ctx->st_ldc, ctx->lse_row, ctx->fac_row,
                            ctx->lse_col, ctx->fac_col, ctx->fac_ok, ctx->st_bad, invN * c_f, 2.f * invN * k.beta_lse,
                            invN * c_b, 0.f, cond, st, ctx->dist ? ctx->st_colsum : nullptr));
      nl += 2;
      if (ctx->dist) {
        // C2: the column sums of e^l over every rank's rows; this rank finalises its own columns
        // (the all-gather below distributes them, as after the two-call path); the fallback
        // gate must agree across ranks (max)
        NC(ncclGroupStart());
        NC(ncclAllReduce(ctx->st_colsum, ctx->st_colsum, (size_t)N, ncclFloat32, ncclSum, ctx->comm, st));
        NC(ncclAllReduce(ctx->st_bad, ctx->st_bad, 1, ncclInt32, ncclMax, ctx->comm, st));
        NC(ncclGroupEnd());
        CU(tc::tc_stats_col_finalize(ctx->st_colsum, row_off, Bl, ctx->lse_col, ctx->fac_col, ctx->fac_ok, ctx->st_bad,
                                     invN * c_b, 0.f, st));
        ++nl;
        NC(ncclAllReduce(ctx->st_bad, ctx->st_bad, 1, ncclInt32, ncclMax, ctx->comm, st));
      }
      gate = ctx->st_bad;
    }
    if (cond != 0) {
      cudaStreamCaptureStatus cs;
      cudaGraph_t cg;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      CU(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = cond;
      np.conditional.type = cudaGraphCondTypeIf;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      CU(cudaGraphAddNode(&node, cg, deps, nd, &np));
      CU(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
      CU(cudaStreamBeginCaptureToGraph(ctx->cap_body, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed));
      CU(tc::tc_logits_lse_pair(D, k.energy, row_side, col_side, Bl, N, S, ctx->fac_ok, ctx->lg_ticket, nullptr,
                                ctx->cap_body));
      cudaGraph_t body_out = nullptr;
      CU(cudaStreamEndCapture(ctx->cap_body, &body_out));
    } else {
    if (std::getenv("CRL_LSE_TWO_CALL")) {   // ablation: the row / column calls on two streams
      fork2(ctx, st, st2);
      { Stage sg(ctx, st2, "lse_col");
        CU(tc::tc_logits_lse(D, k.energy, ctx->lg_col_A, ctx->lg_col_B, Bl, N, ctx->stat_psi + row_off,
                             ctx->stat_phi, S, col_side.part_m, col_side.part_s, ctx->lse_col, ctx->fac_col,
                             ctx->fac_ok, invN * c_b, 0.f, gate, st2));
        nl += 2; }
      { Stage sg(ctx, st, "lse_row");
        CU(tc::tc_logits_lse(D, k.energy, ctx->lg_row_A, ctx->lg_row_B, Bl, N, ctx->stat_phi + row_off,
                             ctx->stat_psi, S, row_side.part_m, row_side.part_s, ctx->lse_row, ctx->fac_row,
                             ctx->fac_ok, invN * c_f, 2.f * invN * k.beta_lse, gate, st));
        nl += 2; }
      join2(ctx, st, st2);
    } else { Stage sg(ctx, st, "lse_pair");
      CU(tc::tc_logits_lse_pair(D, k.energy, row_side, col_side, Bl, N, S, ctx->fac_ok, ctx->lg_ticket, gate, st));
      ++nl; }
    }
  } else {
    if (ctx->dist) {
      NC(ncclGroupStart());
      NC(ncclAllGather(ctx->phi_out, ctx->phi_g, (size_t)Bl * D, ncclFloat32, ctx->comm, st));
      NC(ncclAllGather(ctx->psi_out, ctx->psi_g, (size_t)Bl * D, ncclFloat32, ctx->comm, st));
      NC(ncclGroupEnd());
    }
    fork2(ctx, st, st2);
    { Stage sg(ctx, st2, "lse_col");
      CU(logits_lse_f32(D, k.energy, ctx->psi_out, Bl, ctx->phi_g, N, ctx->lse_col, st2)); ++nl; }
    { Stage sg(ctx, st, "lse_row");
      CU(logits_lse_f32(D, k.energy, ctx->phi_out, Bl, ctx->psi_g, N, ctx->lse_row, st)); ++nl; }
    join2(ctx, st, st2);
  }
  if (ctx->dist) {
    NC(ncclGroupStart());
    NC(ncclAllGather(ctx->lse_row, ctx->lse_row_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
    NC(ncclAllGather(ctx->lse_col, ctx->lse_col_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
    if (ctx->tc_logits) {
      NC(ncclAllGather(ctx->fac_row, ctx->fac_row_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
      NC(ncclAllGather(ctx->fac_col, ctx->fac_col_g, (size_t)Bl, ncclFloat32, ctx->comm, st));
      NC(ncclAllReduce(ctx->fac_ok, ctx->fac_ok, 1, ncclInt32, ncclMin, ctx->comm, st));
    }
    NC(ncclGroupEnd());
  }
  // the loss is reduced inside the fused gradient kernel when that runs (its idle warps)
  tc::GradfLoss gl;
  if (ctx->use_gradf) {
    gl.phi32 = ctx->phi_out; gl.psi32 = ctx->psi_out; gl.part = ctx->loss_part; gl.ticket = ctx->loss_ticket;
    gl.acc = ctx->loss_acc; gl.out = loss_out; gl.skip = ctx->skip; gl.adam_t = ctx->adam_t; gl.status = ctx->status;
    gl.c_f = lsgn * c_f; gl.c_b = lsgn * c_b; gl.beta = k.beta_lse;
  } else if (!ctx->use_grad2) { Stage sg(ctx, st, "loss");
    CU(launch_loss_partial(ctx->phi_out, ctx->psi_out, Bl, D, k.energy, ctx->lse_row, ctx->lse_col,
                           ctx->loss_acc, ctx->loss_part, ctx->loss_ticket, !ctx->dist, invN, lsgn * c_f, lsgn * c_b,
                           k.beta_lse, loss_out, ctx->skip, ctx->adam_t, ctx->status, st));
    ++nl; }
  // (the D = 256 pair gradient path reduces the loss in its merge launch, below)
  if (ctx->dist && !ctx->use_grad2) {
    NC(ncclAllReduce(ctx->loss_acc, ctx->loss_acc, 3, ncclFloat32, ncclSum, ctx->comm, st));
    CU(launch_loss_finalize(ctx->loss_acc, invN, lsgn * c_f, lsgn * c_b, k.beta_lse, loss_out, ctx->skip, ctx->adam_t,
                            ctx->status, st));
    ++nl;
  }
  if (ctx->use_gradf) {
    // both sides of dL/dl from ONE evaluation of every w_ij (tc_gradf.cu); the column side
    // accumulates by reductions into db_acc / cs_acc, zeroed by prep_inputs at the step start
    { Stage sg(ctx, st, "grad_fused");
      CU(tc::tc_grad_fused(k.energy, ctx->lg_row_A, ctx->lg_row_B, ctx->gf_map, Bl, N, ctx->stat_phi, ctx->stat_psi,
                           ctx->lse_row, ctx->lse_col, ctx->fac_col, ctx->fac_ok, c_f, c_b, k.beta_lse, invN,
                           ctx->gf_splits, ctx->gf_part_da, ctx->gf_part_rs, ctx->gf_acc, ctx->gf_cs, ctx->phi_outb,
                           ctx->psi_outb, ctx->dphi, ctx->dphib, ctx->dpsi, ctx->dpsib, gl, st));
      nl += 2; }
  }
  if (ctx->use_grad2) {
    // D = 256: both sides of dL/dl -> dPhi, dPsi in one persistent launch, then one merge
    // launch for both (partial slots, L2 row-sum term, positive pair, cos projection, bf16)
    Stage sg(ctx, st, "grad_pair");
    tc::Grad2Args ga{};
    ga.Na = Bl; ga.Nb = N; ga.invN = invN; ga.fac_ok = ctx->fac_ok;
    tc::Grad2Side& s0 = ga.side[0];
    s0.a_stat = ctx->stat_phi + row_off; s0.b_stat = ctx->stat_psi; s0.lr = ctx->lse_row; s0.lc = ctx->lse_col_g;
    s0.lcf = ctx->fac_col_g; s0.c_r = c_f; s0.c_c = c_b; s0.beta_r = k.beta_lse; s0.beta_c = 0.f;
    s0.part_da = ctx->g2_part_da; s0.part_rs = ctx->g2_part_rs; s0.A = ctx->phi_outb;
    tc::Grad2Side& s1 = ga.side[1];
    s1.a_stat = ctx->stat_psi + row_off; s1.b_stat = ctx->stat_phi; s1.lr = ctx->lse_col; s1.lc = ctx->lse_row_g;
    s1.lcf = ctx->fac_row_g; s1.c_r = c_b; s1.c_c = c_f; s1.beta_r = 0.f; s1.beta_c = k.beta_lse;
    // row-sum sub-slots per partial slot: one per epilogue warpgroup of the launched variant
    const int prs_sub = ctx->g2_pair ? tc::tc_grad2p_warpgroups() : 2;
    s1.part_da = ctx->g2_part_da + (size_t)(ctx->g2_wsym ? 3 : 2) * Bl * D; s1.part_rs = ctx->g2_part_rs + (size_t)2 * prs_sub * Bl;
    s1.A = ctx->psi_outb;
    if (ctx->g2_wsym) { ga.nsides = 1; ga.w_store = 1; }
    if (ctx->g2_pair) CU(tc::tc_grad2p(k.energy, ctx->g2_B0, ctx->g2_B1, ctx->g2_S0, ctx->g2_S1, ctx->g2_A0,
                                           ctx->g2_A1, ga, ctx->g2_grid, st, ctx->g2_wsym ? &ctx->g2_Wmap : nullptr));
    else CU(tc::tc_grad2(k.energy, ctx->g2_B0, ctx->g2_B1, ga, ctx->g2_grid, st));
    // symmetric energies at W = 1: side 1's weights are W^T -> dPsi = W^T Phi (+ column sums of W)
    // on the pair engine (64 items: 10 pairs idle), the row-side merge (+ loss) beside it on st2
    const bool wsym_split = ctx->g2_wsym && st != st2 && !std::getenv("CRL_NO_G2_MERGE_SPLIT");
    if (wsym_split) fork2(ctx, st, st2);
    if (ctx->g2_wsym) { CU(tc::tc_pdw_launch(ctx->pdw_g, ctx->num_sms, st)); ++nl; }
    const float Cdiag = invN * (c_f + c_b);
    tc::GradMergeArgs m0{s0.part_da, s0.part_rs, ctx->phi_outb, s0.a_stat, ctx->psi_outb_g, ctx->stat_psi, row_off,
                         Cdiag, Bl, D, 2, ctx->dphi, ctx->dphib, 0};
    tc::GradMergeArgs m1{s1.part_da, s1.part_rs, ctx->psi_outb, s1.a_stat, ctx->phi_outb_g, ctx->stat_phi, row_off,
                         Cdiag, Bl, D, 2, ctx->dpsi, ctx->dpsib, 0};
    m0.valid1 = ctx->g2_flags;
    m1.valid1 = ctx->g2_flags + (Bl + 127) / 128;
    m0.prs_sub = m1.prs_sub = prs_sub;
    if (ctx->g2_wsym) { m0.S = 3; m1.valid1 = nullptr; m1.prs = ctx->g2_cs; m1.prs_sub = 1; }
    // the loss rides on the row-side merge: l_ii from the bf16 rows the logits used
    tc::MergeLoss ml;
    ml.lr = ctx->lse_row; ml.lc = ctx->lse_col; ml.part = ctx->loss_part; ml.ticket = ctx->loss_ticket;
    ml.acc = ctx->loss_acc; ml.out = loss_out; ml.skip = ctx->skip; ml.adam_t = ctx->adam_t; ml.status = ctx->status;
    ml.invN = invN; ml.c_f = lsgn * c_f; ml.c_b = lsgn * c_b; ml.beta = k.beta_lse; ml.finalize = !ctx->dist;
    if (wsym_split) {
      CU(tc::launch_grad_merge2(k.energy, m0, m0, st2, &ml, 1));
      CU(tc::launch_grad_merge2(k.energy, m1, m1, st, nullptr, 1));
      join2(ctx, st, st2);
      nl += 3;
    } else {
      CU(tc::launch_grad_merge2(k.energy, m0, m1, st, &ml));
      nl += 2;
    }
    if (ctx->dist) {
      NC(ncclAllReduce(ctx->loss_acc, ctx->loss_acc, 3, ncclFloat32, ncclSum, ctx->comm, st));
      CU(launch_loss_finalize(ctx->loss_acc, invN, lsgn * c_f, lsgn * c_b, k.beta_lse, loss_out, ctx->skip,
                              ctx->adam_t, ctx->status, st));
      ++nl;
    }
  }
  fork2(ctx, st, st2);
  if (!ctx->use_gradf && !ctx->use_grad2) { Stage sg(ctx, st2, "grad_psi");
    if (ctx->tc_logits) {
      CU(tc::tc_logits_grad(D, k.energy, ctx->lg_col_A, ctx->lg_col_B, Bl, N, row_off, ctx->stat_psi + row_off,
                            ctx->stat_phi, ctx->lse_col, ctx->lse_row_g, ctx->fac_row_g, c_b, c_f, 0.f,
                            k.beta_lse, invN, S,
                            ctx->lg_part_da + (size_t)S * Bl * D, ctx->lg_part_rs + (size_t)S * Bl,
                            ctx->psi_outb, ctx->phi_outb_g, ctx->dpsi, ctx->dpsib, ctx->fac_ok, st2));
    } else {
      CU(logits_grad_f32(D, k.energy, ctx->psi_out, Bl, row_off, ctx->phi_g, N, ctx->lse_col, ctx->lse_row_g,
                         c_b, c_f, 0.f, k.beta_lse, invN, ctx->dpsi, st2));
      CU(tc::launch_f32_to_bf16(ctx->dpsi, ctx->dpsib, (size_t)Bl * D, ctx->num_sms, st2));
    }
    nl += 2; }
  cudaStream_t side = (st == st2) ? st : ctx->cap_stream3;      // phi weight gradients
  cudaStream_t side2 = (st == st2) ? st : ctx->cap_stream4;     // psi weight gradients
  const bool fused_bwd = ctx->use_chain || ctx->use_cchain;      // one dX-chain launch for both
  // both encoders' dX layers as joint CTA-pair launches (the gradient pass gives dPhi and dPsi at once)
  const bool pair_bwd = !fused_bwd && (ctx->use_pdw || ctx->use_dwg) && (ctx->use_grad2 || ctx->use_gradf) &&
                        pg_pair_layers(ctx, true);
  if (!fused_bwd && !pair_bwd) {
    rs = enc_backward_bf16(ctx, "psi", ctx->psi_plan, ctx->tc_psi, ctx->psiZb, st2, side2, &nl);
    if (rs != CRL_OK) return rs;
  }
  if (!ctx->use_gradf && !ctx->use_grad2) { Stage sg(ctx, st, "grad_phi");
    if (ctx->tc_logits) {
      CU(tc::tc_logits_grad(D, k.energy, ctx->lg_row_A, ctx->lg_row_B, Bl, N, row_off, ctx->stat_phi + row_off,
                            ctx->stat_psi, ctx->lse_row, ctx->lse_col_g, ctx->fac_col_g, c_f, c_b,
                            k.beta_lse, 0.f, invN, S,
                            ctx->lg_part_da, ctx->lg_part_rs, ctx->phi_outb, ctx->psi_outb_g, ctx->dphi,
                            ctx->dphib, ctx->fac_ok, st));
    } else {
      CU(logits_grad_f32(D, k.energy, ctx->phi_out, Bl, row_off, ctx->psi_g, N, ctx->lse_row, ctx->lse_col_g,
                         c_f, c_b, k.beta_lse, 0.f, invN, ctx->dphi, st));
      CU(tc::launch_f32_to_bf16(ctx->dphi, ctx->dphib, (size_t)Bl * D, ctx->num_sms, st));
    }
    nl += 2; }
  if (pair_bwd) {
    join2(ctx, st, st2);
    rs = enc_backward_pair_bf16(ctx, st, &nl);
    if (rs != CRL_OK) return rs;
  } else if (!fused_bwd) {
    rs = enc_backward_bf16(ctx, "phi", ctx->phi_plan, ctx->tc_phi, ctx->phiZb, st, side, &nl);
    if (rs != CRL_OK) return rs;
    join2(ctx, st, st2);
  } else if (ctx->use_chain) {
    join2(ctx, st, st2);
    { Stage sg(ctx, st, "mlp_bwd_chain");          // both encoders' dX chains, one launch
      CU(tc::tc_chain_backward(ctx->chain_bwd[0], ctx->chain_bwd[1], ctx->chain_bwd_p, st));
      ++nl; }
  } else {
    join2(ctx, st, st2);
    { Stage sg(ctx, st, "mlp_bwd_cchain");         // both encoders' dX chains, 4-CTA clusters
      CU(tc::tc_cchain_backward(ctx->cchain_bwd[0], ctx->cchain_bwd[1], ctx->cchain_bwd_p, st));
      ++nl; }
  }
  if (ctx->use_pdw && ctx->pdw_split) {
    // phi's dW / db on st, psi's on st2 (both persistent: psi's pairs start as phi's finish);
    // Adam of each encoder follows its own launch (enqueue_allreduce_adam)
    Stage sg(ctx, st, "dw_db_pairs");
    fork2(ctx, st, st2);
    CU(tc::tc_pdw_launch(ctx->pdw, ctx->num_sms, st));
    CU(tc::tc_pdw_launch(ctx->pdw_psi, ctx->num_sms, st2));
    nl += 2;
  } else if (ctx->use_pdw) {
    // every dW_l and db_l of both encoders on CTA pairs (tc_pdw.cu)
    Stage sg(ctx, st, "dw_db_pairs");
    CU(tc::tc_pdw_launch(ctx->pdw, ctx->num_sms, st));
    ++nl;
  } else if (ctx->use_dwg) {
    // every dW_l and db_l of both encoders in one grouped launch (tc_dwg.cu)
    Stage sg(ctx, st, "dw_db_grouped");
    CU(tc::tc_dwg_launch(ctx->dwg, st));
    ++nl;
  } else if (fused_bwd) {
    if (side != st) {
      cudaEventRecord(ctx->ev_side, st);
      cudaStreamWaitEvent(side, ctx->ev_side, 0);
      cudaStreamWaitEvent(side2, ctx->ev_side, 0);
    }
    rs = enc_weight_grads_bf16(ctx, "phi", ctx->phi_plan, ctx->tc_phi, side, &nl);
    if (rs != CRL_OK) return rs;
    rs = enc_weight_grads_bf16(ctx, "psi", ctx->psi_plan, ctx->tc_psi, side2, &nl);
    if (rs != CRL_OK) return rs;
  }
  if (side != st && !ctx->use_dwg && !ctx->use_pdw) {
    cudaEventRecord(ctx->ev_side, side);
    cudaStreamWaitEvent(st, ctx->ev_side, 0);
    cudaEventRecord(ctx->ev_side, side2);
    cudaStreamWaitEvent(st, ctx->ev_side, 0);
  }
  // A6: Adam; W > 1: split-K partials reduced and the gradient all-reduced in buckets first (C4)
  rs = enqueue_allreduce_adam(ctx, st, st2, ctx->wshadow, grads_out != nullptr, &nl);
  if (rs != CRL_OK) return rs;
  if (grads_out)
    CU(cudaMemcpyAsync(grads_out, ctx->grads, ctx->sizes.n_params * 4, cudaMemcpyDeviceToDevice, st));
  ctx->launches = nl;
  return CRL_OK;
}
