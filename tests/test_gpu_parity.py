"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Tolerances (north_star): relabel indices bit-exact and s/a/g bitwise; fp32 path
loss within 1e-5 relative and gradients within 1e-4 relative (per-tensor L2 norm)."""
import numpy as np
import pytest

import crl_synth
from _crl_testlib import fill_buffer, make_ctx, oracle_buffers, oracle_kw, param_tensors, rel, relmax

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import critic as ocritic       # noqa: E402
from oracle import replay as oreplay       # noqa: E402

SEED = crl_synth.PHILOX_SEED
# element-wise bound, as a multiple of the norm tolerance: max|a - b| / max|b| of a tensor is
# the infinity-norm analogue of the per-tensor L2 check (SURVEY 8(c) parity metric)
EMAX = 3.0


def _sample_gpu(ctx, cfg, step, B=None):
    B = B or ctx.cfg.batch_local
    s = torch.empty(B, cfg["obs_dim"], device="cuda")
    a = torch.empty(B, cfg["act_dim"], device="cuda")
    g = torch.empty(B, cfg["goal_dim"], device="cuda")
    idx = torch.empty(B, 3, dtype=torch.int64, device="cuda")
    ctx.relabel_sample(SEED, step, s, a, g, idx)
    torch.cuda.synchronize()
    return s.cpu().numpy(), a.cpu().numpy(), g.cpu().numpy(), idx.cpu().numpy()


# ------------------------------------------------------------------------- A0 + A1

@pytest.mark.parametrize("name,n_chunks,U,B", [
    ("reacher", 20, 62, 256),      # configs[0]: 8 envs x 1000, ring wrapped (1240 steps)
    ("humanoid", 3, 62, 512),      # configs[2] shapes (obs 268), partially filled ring
    ("reacher", 1, 1, 37),         # degenerate: a single step per env is < 2 slots -> ESTATE
])
def test_relabel_bit_exact(name, n_chunks, U, B):
    cfg = crl_synth.preset(name, precision="fp32", batch=B)
    if name == "humanoid":
        cfg["n_envs"] = 64                      # keep the oracle's Python loops short
    ctx, _ = make_ctx(cfg)
    chunks = fill_buffer(ctx, cfg, n_chunks, U=U)
    if n_chunks * U < 2:
        from paper_2408_11052_b200 import CrlError
        with pytest.raises(CrlError):
            _sample_gpu(ctx, cfg, 0, B)
        return
    bufs = oracle_buffers(cfg, chunks)
    for step in (0, 1, 12345678901):
        s, a, g, idx = _sample_gpu(ctx, cfg, step, B)
        os_, oa, og, oidx = oreplay.relabel_sample(bufs[0], SEED, step, B, gamma=cfg["gamma"],
                                                   goal_offset=cfg["goal_offset"],
                                                   goal_dim=cfg["goal_dim"])
        assert np.array_equal(idx, oidx)
        assert np.array_equal(s.view(np.uint32), os_.view(np.uint32))
        assert np.array_equal(a.view(np.uint32), oa.view(np.uint32))
        assert np.array_equal(g.view(np.uint32), og.view(np.uint32))
    assert ctx.status() == 0


@pytest.mark.parametrize("gamma", [0.0, 0.5, 0.9, 0.999, 0.99999])
def test_relabel_bit_exact_gamma(gamma):
    """The offset lookup (fp64 window estimate + exact integer decision, binary-search
    fallback) across discounts: gamma = 0 (k = 1 always), short and long geometric tails."""
    cfg = crl_synth.preset("reacher", precision="fp32", batch=256)
    cfg["gamma"] = gamma
    ctx, _ = make_ctx(cfg)
    chunks = fill_buffer(ctx, cfg, 20, U=62)
    bufs = oracle_buffers(cfg, chunks)
    for step in (0, 7):
        s, a, g, idx = _sample_gpu(ctx, cfg, step)
        os_, oa, og, oidx = oreplay.relabel_sample(bufs[0], SEED, step, 256, gamma=gamma,
                                                   goal_offset=cfg["goal_offset"],
                                                   goal_dim=cfg["goal_dim"])
        assert np.array_equal(idx, oidx)
        assert np.array_equal(g.view(np.uint32), og.view(np.uint32))
    assert ctx.status() == 0


@pytest.mark.parametrize("alpha", [0.0, 0.37, 1.0])
def test_relabel_random_goal_alpha_bit_exact(alpha):
    """F4 random-goal mixing (App. C, reading A-36): the ACTOR's goals (g_actor of
    crl_relabel_sample_mixed) are bit-exact vs the oracle's random_goal_mix; the critic's g,
    s, a and idx stay the hindsight sample (equal to crl_relabel_sample's, bitwise)."""
    cfg = crl_synth.preset("reacher", precision="fp32", batch=256)
    ctx, _ = make_ctx(cfg, random_goal_alpha=alpha)
    chunks = fill_buffer(ctx, cfg, 20, U=62)
    bufs = oracle_buffers(cfg, chunks)
    B, n = 256, 2
    s = torch.empty(n * B, cfg["obs_dim"], device="cuda")
    a = torch.empty(n * B, cfg["act_dim"], device="cuda")
    g = torch.empty(n * B, cfg["goal_dim"], device="cuda")
    ga = torch.empty(n * B, cfg["goal_dim"], device="cuda")
    idx = torch.empty(n * B, 3, dtype=torch.int64, device="cuda")
    step0 = 9
    ctx.relabel_sample_mixed(SEED, step0, n, s, a, g, ga, idx)
    torch.cuda.synchronize()
    for u in range(n):
        sl = slice(u * B, (u + 1) * B)
        os_, oa, og, oidx = oreplay.relabel_sample(bufs[0], SEED, step0 + u, B, gamma=cfg["gamma"],
                                                   goal_offset=cfg["goal_offset"], goal_dim=cfg["goal_dim"])
        oga, flag = oreplay.random_goal_mix(bufs[0], SEED, step0 + u, B, og, alpha,
                                            goal_offset=cfg["goal_offset"], goal_dim=cfg["goal_dim"])
        assert np.array_equal(idx[sl].cpu().numpy(), oidx)
        assert np.array_equal(s[sl].cpu().numpy().view(np.uint32), os_.view(np.uint32))
        assert np.array_equal(g[sl].cpu().numpy().view(np.uint32), og.view(np.uint32))
        assert np.array_equal(ga[sl].cpu().numpy().view(np.uint32), oga.view(np.uint32))
        if alpha == 1.0:
            assert flag.all()
        elif alpha > 0:
            assert flag.any() and not flag.all()
    assert ctx.status() == 0


def test_relabel_full_size_ant_sampled_rows():
    """configs[1] at full size (1024 envs x 1000, wrapped ring): the oracle recomputes a
    sample of rows one by one."""
    cfg = crl_synth.preset("ant", batch=4096)
    ctx, _ = make_ctx(cfg)
    chunks = fill_buffer(ctx, cfg, 20)
    bufs = oracle_buffers(cfg, chunks)
    s, a, g, idx = _sample_gpu(ctx, cfg, 7)
    rows = list(range(0, 4096, 97)) + [4095]
    _, _, og, oidx = oreplay.relabel_sample(bufs[0], SEED, 7, 4096, gamma=cfg["gamma"],
                                            goal_dim=cfg["goal_dim"], rows=rows)
    assert np.array_equal(idx[rows], oidx[rows])
    assert np.array_equal(g[rows], og[rows])
    # properties over all rows: in-window, strictly future, same episode
    tau_old, tau_new, _ = bufs[0].window()
    assert np.all(idx[:, 1] >= tau_old) and np.all(idx[:, 2] <= tau_new)
    assert np.all(idx[:, 2] > idx[:, 1])


_ANT_ORACLE = {}


def _ant_full_buffers(cfg):
    """configs[1]'s full buffer (1024 envs x 1000, 20 chunks of 62: wrapped), oracle side, built
    once per test session (the GPU side is refilled per context)."""
    if "bufs" not in _ANT_ORACLE:
        chunks = crl_synth.fast_chunks(cfg, 20)
        _ANT_ORACLE["chunks"] = chunks
        _ANT_ORACLE["bufs"] = oracle_buffers(cfg, chunks)
    return _ANT_ORACLE["chunks"], _ANT_ORACLE["bufs"]


@pytest.mark.parametrize("B", [8192, 16384])
@pytest.mark.parametrize("gamma", [0.0, 0.99, 0.99999])
def test_relabel_narrow_path_full_batch_bit_exact(B, gamma):
    """relabel_sample_kernel<4> (4 lanes per row, 8 rows per warp, 4-entry offset window with a
    binary-search fallback) runs for >= 8192 narrow rows (Ant rows: obs 29): every row of the
    sweep8192 / sweep16384 batches compared bit-exactly with the oracle, across discounts
    (gamma = 0: k = 1; 0.99: the paper's; 0.99999: long tails, window misses -> fallback)."""
    cfg = crl_synth.preset("ant", batch=B)
    cfg["gamma"] = gamma
    chunks, bufs = _ant_full_buffers(cfg)
    ctx, _ = make_ctx(cfg)
    for obs, act, done in chunks:
        ctx.buffer_insert(torch.from_numpy(obs).cuda(), torch.from_numpy(act).cuda(), torch.from_numpy(done).cuda())
    s, a, g, idx = _sample_gpu(ctx, cfg, 3)
    os_, oa, og, oidx = oreplay.relabel_sample(bufs[0], SEED, 3, B, gamma=gamma, goal_dim=cfg["goal_dim"])
    assert np.array_equal(idx, oidx)
    assert np.array_equal(s.view(np.uint32), os_.view(np.uint32))
    assert np.array_equal(a.view(np.uint32), oa.view(np.uint32))
    assert np.array_equal(g.view(np.uint32), og.view(np.uint32))
    assert ctx.status() == 0


def test_relabel_bulk_65536_rows_bit_exact():
    """The bench's bulk call (crl_relabel_sample_bulk, 256 updates x B = 256 Ant rows = 65,536
    rows, the <4> kernel): every row equals the oracle's sample at step0 + u, bitwise."""
    cfg = crl_synth.preset("ant", batch=256)
    chunks, bufs = _ant_full_buffers(cfg)
    ctx, _ = make_ctx(cfg)
    for obs, act, done in chunks:
        ctx.buffer_insert(torch.from_numpy(obs).cuda(), torch.from_numpy(act).cuda(), torch.from_numpy(done).cuda())
    n, B, step0 = 256, 256, 41_000_000
    s = torch.empty(n * B, cfg["obs_dim"], device="cuda")
    a = torch.empty(n * B, cfg["act_dim"], device="cuda")
    g = torch.empty(n * B, cfg["goal_dim"], device="cuda")
    idx = torch.empty(n * B, 3, dtype=torch.int64, device="cuda")
    ctx.relabel_sample_bulk(SEED, step0, n, s, a, g, idx)
    torch.cuda.synchronize()
    s, a, g, idx = (x.cpu().numpy() for x in (s, a, g, idx))
    for u in range(n):
        sl = slice(u * B, (u + 1) * B)
        os_, oa, og, oidx = oreplay.relabel_sample(bufs[0], SEED, step0 + u, B, gamma=cfg["gamma"],
                                                   goal_dim=cfg["goal_dim"])
        assert np.array_equal(idx[sl], oidx), u
        assert np.array_equal(s[sl].view(np.uint32), os_.view(np.uint32)), u
        assert np.array_equal(a[sl].view(np.uint32), oa.view(np.uint32)), u
        assert np.array_equal(g[sl].view(np.uint32), og.view(np.uint32)), u
    assert ctx.status() == 0


# ------------------------------------------------------------------------- A2-A6

def _critic_parity(cfg, batch_seed=11, check_adam=True, tol_loss=1e-5, tol_grad=1e-4, per_layer=True,
                   encoder_grads=True):
    ctx, params = make_ctx(cfg)
    B = cfg["batch"]
    s, a, g = crl_synth.random_batch(cfg, B, seed=batch_seed)
    loss = torch.zeros(4, device="cuda")
    grads = torch.zeros(ctx.n_params, device="cuda")
    ctx.critic_step(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(),
                    torch.from_numpy(g).cuda(), loss, grads)
    torch.cuda.synchronize()
    assert ctx.status() == 0
    z = np.zeros_like(params, dtype=np.float64)
    ref = ocritic.critic_step(params.astype(np.float64), z, z, 0, s, a, g, lr=cfg["lr"],
                              **oracle_kw(cfg))
    L = loss.cpu().numpy()
    for i, k in enumerate(["L_fwd", "L_bwd", "penalty", "total"]):
        assert abs(L[i] - ref[k]) <= tol_loss * max(abs(ref[k]), 1e-3), (k, L[i], ref[k])
    assert rel(ctx.debug_tensor("phi").cpu().numpy(), ref["phi"]) < tol_loss
    assert rel(ctx.debug_tensor("lse_row").cpu().numpy(), ref["lse_row"]) < tol_loss
    assert rel(ctx.debug_tensor("lse_col").cpu().numpy(), ref["lse_col"]) < tol_loss
    for name in ("dphi", "dpsi"):
        got = ctx.debug_tensor(name).cpu().numpy()
        assert rel(got, ref[name]) < tol_grad, name
        assert relmax(got, ref[name]) < EMAX * tol_grad, (name, relmax(got, ref[name]))
    if not encoder_grads:
        return
    gr = grads.cpu().numpy()
    assert rel(gr, ref["grads"]) < tol_grad
    # per-tensor (every W, b and LayerNorm gamma / beta: a wrong small tensor can hide in the
    # global norm), in the L2 norm and element by element (max |a - b| / max |b|)
    off = 0
    for name, n in param_tensors(cfg):
        if per_layer:
            assert rel(gr[off:off + n], ref["grads"][off:off + n]) < tol_grad, name
            em = relmax(gr[off:off + n], ref["grads"][off:off + n])
            assert em < EMAX * tol_grad, (name, em)
        off += n
    assert off == gr.size
    if check_adam:
        # The first Adam step maps g -> g/(|g|+eps) ~ sign(g): it magnifies tiny gradient
        # differences near |g| ~ eps, so the optimiser kernel is checked on the GPU's own
        # gradients (oracle Adam, fp64) and the end-to-end delta only loosely.
        from oracle import adam as oadam
        dp = ctx.params.cpu().numpy().astype(np.float64) - params
        p_ref, *_ = oadam.adam_step(params.astype(np.float64), gr.astype(np.float64), z, z, 0,
                                    lr=cfg["lr"])
        # the parameters are stored in fp32: round the oracle's update the same way (for
        # parameters near 1, e.g. LayerNorm gains, one fp32 ulp is ~4e-4 of a 3e-4 step)
        assert rel(dp, p_ref.astype(np.float32).astype(np.float64) - params) < 1e-5
        if tol_grad <= 1e-4:
            assert rel(dp, ref["params_new"] - params) < 1e-2
    return ctx


@pytest.mark.parametrize("energy", ["l2", "dot", "cos"])
@pytest.mark.parametrize("loss", ["fwd", "bwd", "sym"])
def test_critic_step_fp32_small(energy, loss):
    cfg = crl_synth.preset("reacher", batch=200, width=64, energy=energy, loss=loss)
    _critic_parity(cfg)


@pytest.mark.parametrize("energy", ["l1", "l2sq"])
@pytest.mark.parametrize("loss", ["fwd", "bwd", "sym"])
def test_critic_step_fp32_f3_energies(energy, loss):
    """L1 and L2-without-sqrt energies (App. A.2) on the fp32
    path, same bar as the other energies (ragged batch, several column tiles)."""
    cfg = crl_synth.preset("reacher", batch=200, width=64, energy=energy, loss=loss)
    _critic_parity(cfg)


def test_critic_step_f3_energies_repr256_ant():
    cfg = crl_synth.preset("ant", precision="fp32", batch=130, repr_dim=256, energy="l1")
    _critic_parity(cfg)


def test_l1_energy_bf16_unsupported():
    """L1 is not a contraction (no tensor-core form): a bf16 context with it is refused."""
    from paper_2408_11052_b200 import CrlError
    cfg = crl_synth.preset("reacher", precision="bf16", batch=64, energy="l1")
    with pytest.raises(CrlError):
        make_ctx(cfg)


@pytest.mark.parametrize("batch,width,repr_dim,knob", [
    (256, 128, 64, None),                    # SIMT logits (N < 1024)
    (1100, 128, 64, None),                   # tensor-core logits, one-pass statistics, two-call gradient
    (1100, 128, 64, "CRL_NO_FUSED_STATS"),   # two-call online-max statistics
    (1100, 128, 64, "CRL_FORCE_EXACT_Q"),
    (1100, 256, 256, None),                  # D = 256: CTA-pair both-sides gradient pass
    (2900, 256, 256, "CRL_NO_GRAD2P"),       # single-CTA both-sides pass
    (1100, 256, 256, "CRL_NO_GRAD2"),
])
def test_critic_step_bf16_l2sq(batch, width, repr_dim, knob, monkeypatch):
    """SURVEY 8(f) F3 L2-without-sqrt energy (App. A.2) on the bf16 tensor-core path:
    l_ij = -max(|a|^2 + |b|^2 - 2 a.b, 0) from the same contraction as L2, w_ij = 2 g_ij."""
    if knob:
        monkeypatch.setenv(knob, "1")
    cfg = crl_synth.preset("ant", batch=batch, width=width, repr_dim=repr_dim, energy="l2sq", precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("loss", ["fwd", "bwd", "sym"])
def test_critic_step_bf16_l2sq_losses(loss):
    cfg = crl_synth.preset("ant", batch=1100, width=128, energy="l2sq", loss=loss, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("act", ["silu", "relu"])
def test_critic_step_fp32_layernorm_small(act):
    """F2 LayerNorm encoders (reading A-35) on the fp32 path: ragged batch, 3 hidden layers."""
    cfg = crl_synth.preset("reacher", batch=150, width=96, depth=3, activation=act, layernorm=1)
    _critic_parity(cfg)


def test_critic_step_fp32_layernorm_netscale_width():
    """The paper's LayerNorm network: 4 x 1024 encoders, repr 256 (config 5 shapes), a batch
    the fp64 oracle finishes quickly."""
    cfg = crl_synth.preset("netscale", precision="fp32", batch=192, layernorm=1)
    _critic_parity(cfg)


def test_layernorm_bf16_unsupported():
    """bf16 LayerNorm needs CTA-pair GEMMs for every hidden layer: width in {256, ..., 1024}
    (a multiple of 256) and at least 256 rows; narrower shapes are refused, not approximated."""
    from paper_2408_11052_b200 import CrlError
    cfg = crl_synth.preset("reacher", precision="bf16", batch=64, layernorm=1)
    with pytest.raises(CrlError):
        make_ctx(cfg)


# SiLU (reading A-13, the default).  ReLU with bf16 operands flips act' = 1[y > 0] for the
# pre-activations bf16 rounding moves across 0, and the flips compound toward the first layer
# (measured: first-layer dW error 4.5 % without and 8.9 % with LN at width 512, B = 512 --
# operand rounding, not a kernel error: the SiLU runs of the same kernels stay below 1.1 %).
@pytest.mark.parametrize("preset,batch,width", [
    ("netscale", 300, 1024),    # the paper's LN network (4 x 1024, repr 256), ragged pair tile
    ("ant", 512, 512),          # width 512, repr 64
    ("ant", 640, 256),          # width 256 (one N tile per layer)
])
def test_critic_step_bf16_layernorm(preset, batch, width):
    """F2 LayerNorm encoders on the bf16 tensor-core path (ln.cu bf16 kernels around the
    CTA-pair GEMMs: Z -> LN -> act forward, act' at Y in the dX epilogue, dY -> dZ plus the
    dgamma / dbeta CTA partials backward) against the fp64 oracle, per tensor incl. gamma, beta."""
    cfg = crl_synth.preset(preset, precision="bf16", batch=batch, width=width, layernorm=1)
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("B", [2, 3, 65, 130])
def test_critic_step_fp32_ragged(B):
    cfg = crl_synth.preset("reacher", batch=B, width=96, depth=3, beta_lse=0.0)
    _critic_parity(cfg)


def test_critic_step_fp32_relu_and_beta():
    cfg = crl_synth.preset("ant", batch=128, width=128, activation="relu", beta_lse=0.5)
    _critic_parity(cfg)


@pytest.mark.parametrize("name", ["reacher", "ant"])
def test_critic_step_fp32_paper_configs(name):
    """configs[0] and configs[1] at their full sizes (batch 256, 2x256 / 4x256)."""
    _critic_parity(crl_synth.preset(name))


def test_critic_step_fp32_repr256():
    cfg = crl_synth.preset("ant", batch=192, width=128, repr_dim=256, precision="fp32")
    _critic_parity(cfg)


def test_critic_step_fp32_sweep4096():
    """configs[3] at batch 4096 (the bench launch configuration)."""
    _critic_parity(crl_synth.preset("sweep4096"), check_adam=False)


def test_critic_step_graph_replay_and_host_buffers():
    """Two steps: the second replays the cached graph; host (pinned) batch + host loss go
    through the end-to-end path.  Compared with two oracle steps."""
    cfg = crl_synth.preset("reacher", batch=96, width=64)
    ctx, params = make_ctx(cfg)
    s, a, g = crl_synth.random_batch(cfg, 96, seed=3)
    sd, ad, gd = (torch.from_numpy(x).cuda() for x in (s, a, g))
    loss_d = torch.zeros(4, device="cuda")
    ctx.critic_step(sd, ad, gd, loss_d)
    s2, a2, g2 = crl_synth.random_batch(cfg, 96, seed=4)
    hs, ha, hg = (torch.from_numpy(x).pin_memory() for x in (s2, a2, g2))
    loss_h = torch.zeros(4).pin_memory()
    ctx.critic_step(hs, ha, hg, loss_h)
    torch.cuda.synchronize()
    kw = oracle_kw(cfg)
    z = np.zeros_like(params, dtype=np.float64)
    r1 = ocritic.critic_step(params.astype(np.float64), z, z, 0, s, a, g, lr=cfg["lr"], **kw)
    r2 = ocritic.critic_step(r1["params_new"], r1["m_new"], r1["v_new"], r1["t_new"], s2, a2, g2,
                             lr=cfg["lr"], **kw)
    assert abs(loss_d.cpu().numpy()[3] - r1["total"]) < 1e-5 * abs(r1["total"])
    assert abs(loss_h.numpy()[3] - r2["total"]) < 1e-5 * abs(r2["total"])
    dp = ctx.params.cpu().numpy().astype(np.float64) - params
    assert rel(dp, r2["params_new"] - params) < 1e-3
    assert ctx.launch_count() > 0


@pytest.mark.parametrize("zero_copy", [True, False])
def test_critic_step_bf16_host_buffers(zero_copy, monkeypatch):
    """bf16 path with page-locked host s, a, g (staged by copies) and a host loss written in
    place by the loss kernel (zero copy) or copied back (CRL_NO_ZERO_COPY) -- both equal the
    device-buffer run of the same batch bitwise (same kernels, same inputs)."""
    if not zero_copy:
        monkeypatch.setenv("CRL_NO_ZERO_COPY", "1")
    cfg = crl_synth.preset("ant", batch=256, precision="bf16")
    s, a, g = crl_synth.random_batch(cfg, 256, seed=8)
    ctx_d, _ = make_ctx(cfg)
    loss_d = torch.zeros(4, device="cuda")
    ctx_d.critic_step(*(torch.from_numpy(x).cuda() for x in (s, a, g)), loss_d)
    ctx_h, _ = make_ctx(cfg)
    hs, ha, hg = (torch.from_numpy(x).pin_memory() for x in (s, a, g))
    loss_h = torch.zeros(4).pin_memory()
    for _ in range(2):                               # second call replays the captured graph
        ctx_h.critic_step(hs, ha, hg, loss_h)
        torch.cuda.synchronize()
        if _ == 0:
            first = loss_h.numpy().copy()
    assert np.array_equal(first.view(np.uint32), loss_d.cpu().numpy().view(np.uint32))
    assert np.isfinite(loss_h.numpy()).all() and ctx_h.status() == 0


def test_critic_step_nonfinite_sets_status_and_skips_adam():
    cfg = crl_synth.preset("reacher", batch=64, width=32)
    ctx, params = make_ctx(cfg)
    s, a, g = crl_synth.random_batch(cfg, 64)
    s[3, 0] = np.nan
    ctx.critic_step(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(), torch.from_numpy(g).cuda())
    torch.cuda.synchronize()
    assert ctx.status(reset=True) == 5          # CRL_ENONFINITE
    assert np.array_equal(ctx.params.cpu().numpy(), params)


# ------------------------------------------------------------------------- BF16 tensor-core path
BF16_TOL = 2e-2          # north_star: bf16 path within 2e-2 relative of the oracle


@pytest.mark.parametrize("energy", ["l2", "dot", "cos"])
def test_critic_step_bf16_small(energy):
    cfg = crl_synth.preset("ant", batch=256, width=128, energy=energy, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("B", [2, 130, 300])
def test_critic_step_bf16_ragged(B):
    cfg = crl_synth.preset("reacher", batch=B, width=64, depth=3, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


def test_critic_step_bf16_humanoid_config():
    """configs[2] at full size: Humanoid shapes (obs 268 + act 17 = 285 inputs), 4x256,
    batch 512, bf16 tensor-core path."""
    _critic_parity(crl_synth.preset("humanoid"), tol_loss=BF16_TOL, tol_grad=BF16_TOL)


def test_critic_step_bf16_sweep4096():
    _critic_parity(crl_synth.preset("sweep4096", precision="bf16"), check_adam=False,
                   tol_loss=BF16_TOL, tol_grad=BF16_TOL)


def test_critic_step_bf16_repr256_width1024():
    """configs[4] network shapes (4x1024, repr 256) at a batch the oracle finishes quickly."""
    cfg = crl_synth.preset("netscale", batch=512)
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


# tensor-core logits stage (bf16 path, N >= 1024): ragged N (not a multiple of the 128-row
# tiles), every energy and loss kind, D = 64 and D = 256
@pytest.mark.parametrize("energy", ["l2", "dot", "cos"])
@pytest.mark.parametrize("loss", ["fwd", "bwd", "sym"])
def test_critic_step_bf16_tc_logits(energy, loss):
    cfg = crl_synth.preset("ant", batch=1100, width=128, energy=energy, loss=loss, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("loss", ["flatnce_fwd", "flatnce_bwd"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_critic_step_flatnce(loss, precision):
    """F3 FlatNCE (reading A-24): InfoNCE gradient, reported L_fwd = L_bwd = 0 and total =
    the logsumexp penalty, on both precisions."""
    if precision == "fp32":
        cfg = crl_synth.preset("reacher", batch=200, width=64, loss=loss)
        _critic_parity(cfg)
    else:
        cfg = crl_synth.preset("ant", batch=1100, width=128, loss=loss, precision="bf16")
        _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("loss", ["fb", "dpo", "ipo", "sppo"])
@pytest.mark.parametrize("energy", ["l2", "dot", "cos", "l1", "l2sq"])
def test_critic_step_fp32_pair_losses(loss, energy):
    """F3 FB / DPO / IPO / SPPO on the fp32 path: ragged batch over several column
    tiles, logsumexp penalty on."""
    cfg = crl_synth.preset("reacher", batch=150, width=64, energy=energy, loss=loss)
    if loss == "fb" and energy == "dot":
        cfg["beta_lse"] = 0.0
    _critic_parity(cfg)


@pytest.mark.parametrize("loss", ["fb", "sppo"])
def test_pair_losses_bf16_or_dp_unsupported(loss):
    from paper_2408_11052_b200 import CrlError
    cfg = crl_synth.preset("reacher", precision="bf16", batch=64, loss=loss)
    with pytest.raises(CrlError):
        make_ctx(cfg)


def _blockwise_lse(kind, Phi, Psi, block=512):
    """Row and column logsumexps of the N x N oracle logits (oracle/energy.py, difference form)
    computed one row block at a time (the N x N matrix never exists in full; blocks run on a
    thread pool: NumPy releases the GIL in its loops).  Columns: an online (max, sum) merge."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    from oracle import energy as oenergy
    from oracle import losses as olosses
    N = Phi.shape[0]

    def one(r0):
        L = oenergy.logits(kind, Phi[r0:r0 + block], Psi)
        m = L.max(0)
        return r0, olosses.lse_rows(L), m, np.exp(L - m[None, :]).sum(0)

    lse = np.empty(N)
    cm = np.full(N, -np.inf)
    cs = np.zeros(N)
    with ThreadPoolExecutor(max(1, len(os.sched_getaffinity(0)))) as ex:
        for r0, lr, m, sm in ex.map(one, range(0, N, block)):
            lse[r0:r0 + block] = lr
            mm = np.maximum(cm, m)
            cs = cs * np.exp(cm - mm) + sm * np.exp(m - mm)
            cm = mm
    return lse, cm + np.log(cs)


def _blockwise_dreps(kind, loss_kind, beta, Phi, Psi, lse, lsec, block=512):
    """dPhi and dPsi of the whole batch through the oracle's row-gradient formula and energy VJP,
    one row block at a time (dPsi summed over the blocks)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    from oracle import energy as oenergy
    from oracle import losses as olosses
    N = Phi.shape[0]

    def one(r0):
        rows = np.arange(r0, min(N, r0 + block))
        L = oenergy.logits(kind, Phi[rows], Psi)
        G = olosses.grad_rows(L, rows, lse, lsec, loss_kind, beta)
        dphi, dpsi = oenergy.vjp(kind, Phi[rows], Psi, G)
        return r0, dphi, dpsi

    dPhi = np.empty_like(Phi)
    dPsi = np.zeros_like(Psi)
    with ThreadPoolExecutor(max(1, len(os.sched_getaffinity(0)))) as ex:
        for r0, dphi, dpsi in ex.map(one, range(0, N, block)):
            dPhi[r0:r0 + block] = dphi
            dPsi += dpsi
    return dPhi, dPsi


@pytest.mark.parametrize("preset,energy", [("sweep16384", None), ("sweep16384", "cos"), ("netscale", None)])
def test_critic_step_bf16_full_size_sampled(preset, energy):
    """configs[3] at its largest batch and configs[4] (4 x 1024, D 256) at full size, in the
    launch configuration bench.py times (one critic step through the C ABI).  Against the fp64
    oracle at the bf16 bar (2e-2):
      * sampled phi / psi rows, every row and column logsumexp (blockwise oracle pass over the
        N x N logits), and the four loss components;
      * sampled dPhi_i / dPsi_j rows (oracle row-gradient formula + energy VJP per row);
      * sweep16384 (L2, the benched energy): the WHOLE pre-Adam gradient, every W and b of both
        encoders, from the oracle's encoder backward fed with blockwise dPhi / dPsi."""
    from oracle import energy as oenergy
    from oracle import losses as olosses
    from oracle import mlp as omlp
    cfg = crl_synth.preset(preset, precision="bf16", **({"energy": energy} if energy else {}))
    N = cfg["batch"]
    ctx, params = make_ctx(cfg)
    s, a, g = crl_synth.random_batch(cfg, N, seed=13)
    loss = torch.zeros(4, device="cuda")
    grads = torch.zeros(ctx.n_params, device="cuda")
    ctx.critic_step(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(), torch.from_numpy(g).cuda(), loss, grads)
    torch.cuda.synchronize()
    assert ctx.status() == 0
    phi_l, psi_l = ocritic.split_critic_params(params.astype(np.float64), cfg["obs_dim"], cfg["act_dim"],
                                               cfg["goal_dim"], cfg["depth"], cfg["width"], cfg["repr_dim"])
    Phi, cache_phi = omlp.forward(phi_l, np.concatenate([s, a], axis=1).astype(np.float64), cfg["activation"])
    Psi, cache_psi = omlp.forward(psi_l, g.astype(np.float64), cfg["activation"])
    rows = np.random.default_rng(5).choice(N, 48, replace=False)
    gphi = ctx.debug_tensor("phi").cpu().numpy().reshape(N, -1)
    gpsi = ctx.debug_tensor("psi").cpu().numpy().reshape(N, -1)
    glr = ctx.debug_tensor("lse_row").cpu().numpy()
    glc = ctx.debug_tensor("lse_col").cpu().numpy()
    for i in rows:
        assert rel(gphi[i], Phi[i]) < BF16_TOL, i
        assert rel(gpsi[i], Psi[i]) < BF16_TOL, i
    lse, lsec = _blockwise_lse(cfg["energy"], Phi, Psi)
    assert np.all(np.abs(glr - lse) <= BF16_TOL * np.maximum(1.0, np.abs(lse)))
    assert np.all(np.abs(glc - lsec) <= BF16_TOL * np.maximum(1.0, np.abs(lsec)))
    # the loss (C4): L_fwd, L_bwd, penalty, total from the oracle's statistics and positives
    diag = oenergy.diag_logits(cfg["energy"], Phi, Psi)
    Lf, Lb = np.mean(lse - diag), np.mean(lsec - diag)
    P = cfg["beta_lse"] * np.mean(lse ** 2)
    ref = {"L_fwd": Lf, "L_bwd": Lb, "penalty": P, "total": Lf + Lb + P}
    Lg = loss.cpu().numpy()
    for k_, key in enumerate(["L_fwd", "L_bwd", "penalty", "total"]):
        assert abs(Lg[k_] - ref[key]) <= BF16_TOL * abs(ref[key]), (key, Lg[k_], ref[key])
    # sampled gradient rows
    gdphi = ctx.debug_tensor("dphi").cpu().numpy().reshape(N, -1)
    gdpsi = ctx.debug_tensor("dpsi").cpu().numpy().reshape(N, -1)
    for i in rows[:16]:
        Lr = oenergy.logits(cfg["energy"], Phi[i:i + 1], Psi)
        Gr = olosses.grad_rows(Lr, [i], lse, lsec, cfg["loss"], cfg["beta_lse"])
        dphi_i, _ = oenergy.vjp(cfg["energy"], Phi[i:i + 1], Psi, Gr)
        assert rel(gdphi[i], dphi_i[0]) < BF16_TOL, (i, rel(gdphi[i], dphi_i[0]))
        # column j = i: the same formula on the transposed problem (rows <-> columns)
        Lc = oenergy.logits(cfg["energy"], Psi[i:i + 1], Phi)
        kind_t = {"fwd": "bwd", "bwd": "fwd"}.get(cfg["loss"], cfg["loss"])
        Gc = olosses.grad_rows(Lc, [i], lsec, lse, kind_t, 0.0)
        # the penalty acts on row LSEs only: its column-side term is (2 beta / N) LSE_k p_k,j
        Gc = Gc + (2.0 * cfg["beta_lse"] / N) * (lse * np.exp(Lc[0] - lse))[None, :]
        dpsi_i, _ = oenergy.vjp(cfg["energy"], Psi[i:i + 1], Phi, Gc)
        assert rel(gdpsi[i], dpsi_i[0]) < BF16_TOL, (i, rel(gdpsi[i], dpsi_i[0]))
    if preset != "sweep16384" or cfg["energy"] != "l2":
        return
    # the whole pre-Adam gradient at N = 16,384 (BASELINE.md §4 allows one oracle step here)
    dPhi, dPsi = _blockwise_dreps(cfg["energy"], cfg["loss"], cfg["beta_lse"], Phi, Psi, lse, lsec)
    assert rel(gdphi, dPhi) < BF16_TOL and rel(gdpsi, dPsi) < BF16_TOL
    g_phi, _ = omlp.backward(phi_l, cache_phi, dPhi, cfg["activation"])
    g_psi, _ = omlp.backward(psi_l, cache_psi, dPsi, cfg["activation"])
    ref_g = np.concatenate([omlp.pack(g_phi), omlp.pack(g_psi)])
    gr = grads.cpu().numpy()
    assert gr.size == ref_g.size
    assert rel(gr, ref_g) < BF16_TOL
    off = 0
    for name, n in param_tensors(cfg):
        assert rel(gr[off:off + n], ref_g[off:off + n]) < BF16_TOL, (name, rel(gr[off:off + n], ref_g[off:off + n]))
        off += n


def energy_row(kind, x, Y):
    """f(x, y_j) for every row y_j of Y (oracle/energy.py, one row at a time)."""
    from oracle import energy as oenergy
    return oenergy.logits(kind, x[None, :], Y)[0]


def logsumexp(v):
    m = v.max()
    return m + np.log(np.exp(v - m).sum())


def test_critic_step_bf16_tc_logits_repr256():
    cfg = crl_synth.preset("ant", batch=1536, width=128, repr_dim=256, precision="bf16", beta_lse=0.3)
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("preset,over", [
    ("ant", dict(batch=256, energy="l2")),
    ("ant", dict(batch=300, energy="cos")),                          # ragged last row block
    ("reacher", dict(batch=130, width=64, depth=3, energy="dot")),   # N = 64 layers, one chunk
    ("humanoid", dict()),                                           # 285 inputs: 5 K chunks
    ("sweep4096", dict()),
])
def test_critic_step_bf16_fused_chain(preset, over, monkeypatch):
    """The fused per-row-block MLP chain kernels (all layers of both encoders in one launch,
    forward and dX backward) are the default only from B_l = 8192; force them here."""
    monkeypatch.setenv("CRL_CHAIN", "1")
    cfg = crl_synth.preset(preset, precision="bf16", **over)
    _critic_parity(cfg, check_adam=cfg["batch"] <= 1024, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("knob,energy", [
    ("CRL_FORCE_STATS_FALLBACK", "l2"),   # fused pass runs, its merge flags, exact pass redoes it
    ("CRL_FORCE_STATS_FALLBACK", "cos"),
    ("CRL_NO_FUSED_STATS", "l2"),         # two-call online-max statistics only
    ("CRL_NO_FUSED_GRAD", "l2"),          # two-call gradient pass (row call + column call)
    ("CRL_NO_FUSED_GRAD", "dot"),
    ("CRL_NO_FUSED_GRAD", "cos"),
    ("CRL_FORCE_STATS_FALLBACK,CRL_COND_NODE", "l2"),   # fallback as a conditional graph node
])
def test_critic_step_bf16_stats_paths(knob, energy, monkeypatch):
    """The one-pass row+column statistics (tc_stats.cu) are the default for L2 / cos at W = 1;
    its exact fallback (taken when a sum under/overflows) and the two-call path are forced."""
    for kn in knob.split(","):
        monkeypatch.setenv(kn, "1")
    cfg = crl_synth.preset("ant", batch=1100, width=128, energy=energy, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("chain", [False, True])
def test_critic_step_bf16_relu(chain, monkeypatch):
    """ReLU on the bf16 path: loss and the global gradient hold the 2e-2 bar; the per-tensor
    check does not apply (reading A-28: bf16 rounding of Z flips ReLU masks near 0,
    and an fp64 emulation of the bf16 operand rounding alone already puts the first phi
    layer's dW ~6% from the fp64 oracle, while SiLU stays at ~0.5%)."""
    if chain:
        monkeypatch.setenv("CRL_CHAIN", "1")
    cfg = crl_synth.preset("ant", batch=300, energy="cos", activation="relu", precision="bf16")
    _critic_parity(cfg, check_adam=False, tol_loss=BF16_TOL, tol_grad=BF16_TOL, per_layer=False)


@pytest.mark.parametrize("energy", ["l2", "cos"])
def test_critic_step_bf16_tc_logits_exact_q_path(energy, monkeypatch):
    """The gradient pass normally forms q_ij = p_ij 2^lse2_i 2^-lse2'_j; the exact second-exp2
    path (taken when a factor is not a normal float) is forced here and checked the same way."""
    monkeypatch.setenv("CRL_FORCE_EXACT_Q", "1")
    cfg = crl_synth.preset("ant", batch=1100, width=128, energy=energy, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


def test_relabel_bulk_matches_single_calls_and_oracle():
    """F4 bulk sampling: row u*B + r equals row r of the single call at step0 + u (bitwise)
    and the oracle's sample at that step."""
    cfg = crl_synth.preset("reacher", precision="fp32", batch=96)
    ctx, _ = make_ctx(cfg)
    chunks = fill_buffer(ctx, cfg, 20, U=62)
    bufs = oracle_buffers(cfg, chunks)
    n, B, step0 = 5, 96, 2 ** 32 - 2                  # the step crosses the 32-bit boundary
    s = torch.empty(n * B, cfg["obs_dim"], device="cuda")
    a = torch.empty(n * B, cfg["act_dim"], device="cuda")
    g = torch.empty(n * B, cfg["goal_dim"], device="cuda")
    idx = torch.empty(n * B, 3, dtype=torch.int64, device="cuda")
    ctx.relabel_sample_bulk(SEED, step0, n, s, a, g, idx)
    torch.cuda.synchronize()
    for u in range(n):
        s1, a1, g1, i1 = _sample_gpu(ctx, cfg, step0 + u)
        sl = slice(u * B, (u + 1) * B)
        assert np.array_equal(idx[sl].cpu().numpy(), i1)
        assert np.array_equal(s[sl].cpu().numpy().view(np.uint32), s1.view(np.uint32))
        assert np.array_equal(a[sl].cpu().numpy().view(np.uint32), a1.view(np.uint32))
        assert np.array_equal(g[sl].cpu().numpy().view(np.uint32), g1.view(np.uint32))
        if u in (0, n - 1):
            _, _, og, oidx = oreplay.relabel_sample(bufs[0], SEED, step0 + u, B, gamma=cfg["gamma"],
                                                    goal_offset=cfg["goal_offset"], goal_dim=cfg["goal_dim"])
            assert np.array_equal(i1, oidx)
            assert np.array_equal(g1.view(np.uint32), og.view(np.uint32))
    from paper_2408_11052_b200 import CrlError
    with pytest.raises(CrlError):
        ctx.relabel_sample_bulk(SEED, 0, 0, s, a, g)
    assert ctx.status() == 0


@pytest.mark.parametrize("energy,knob", [("dot", None), ("l2", "CRL_FORCE_STATS_FALLBACK")])
def test_lse_pair_ticket_rearms_across_steps(energy, knob, monkeypatch):
    """The two-sided statistics launch merges each row block in-kernel by its last split CTA
    (ticket counters left at zero).  With a negligible lr the parameters stay fixed, so every replay
    of the captured step must reproduce the oracle's row and column logsumexps (lr = 1e-12:
    the Adam steps stay below one fp32 ulp of the weights)."""
    if knob:
        monkeypatch.setenv(knob, "1")
    cfg = crl_synth.preset("ant", batch=1100, width=128, energy=energy, precision="bf16", lr=1e-12)
    ctx, params = make_ctx(cfg)
    s, a, g = crl_synth.random_batch(cfg, cfg["batch"], seed=21)
    z = np.zeros_like(params, dtype=np.float64)
    ref = ocritic.critic_step(params.astype(np.float64), z, z, 0, s, a, g, lr=1e-12, **oracle_kw(cfg))
    st, at, gt = (torch.from_numpy(x).cuda() for x in (s, a, g))
    loss = torch.zeros(4, device="cuda")
    for _ in range(4):
        ctx.critic_step(st, at, gt, loss)
        torch.cuda.synchronize()
        assert ctx.status() == 0
        assert rel(ctx.debug_tensor("lse_row").cpu().numpy(), ref["lse_row"]) < BF16_TOL
        assert rel(ctx.debug_tensor("lse_col").cpu().numpy(), ref["lse_col"]) < BF16_TOL
        assert abs(loss[3].item() - ref["total"]) <= BF16_TOL * abs(ref["total"])


def test_critic_step_bf16_ant_config():
    """configs[1] exactly as `bench.py --workload ant` times it (B = 256, 4 x 256, repr 64, L2,
    symmetric InfoNCE, beta 0.1, bf16 tensor-core path with the cluster-chain encoders)."""
    _critic_parity(crl_synth.preset("ant", precision="bf16"), tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("B", [97, 255])
def test_critic_step_bf16_host_buffers_odd_batch(B):
    """Host (page-locked) batches whose s / a / g byte sizes are not multiples of 16 (odd B,
    goal_dim 2): every slot of the host staging ring must stay 16-byte aligned (the device pulls
    it with 16-byte loads).  Several calls walk the ring; each equals the device-buffer run."""
    cfg = crl_synth.preset("reacher", batch=B, precision="bf16")
    ctx_h, _ = make_ctx(cfg)
    ctx_d, _ = make_ctx(cfg)
    for it in range(6):
        s, a, g = crl_synth.random_batch(cfg, B, seed=100 + it)
        loss_d = torch.zeros(4, device="cuda")
        ctx_d.critic_step(*(torch.from_numpy(x).cuda() for x in (s, a, g)), loss_d)
        hs, ha, hg = (torch.from_numpy(x).pin_memory() for x in (s, a, g))
        loss_h = torch.zeros(4).pin_memory()
        ctx_h.critic_step(hs, ha, hg, loss_h)
        torch.cuda.synchronize()
        assert ctx_h.status() == 0 and ctx_d.status() == 0
        assert np.array_equal(loss_h.numpy().view(np.uint32), loss_d.cpu().numpy().view(np.uint32)), it


def test_graph_cache_is_bounded_and_exact():
    """crl_critic_step captures one CUDA graph per pointer tuple into a bounded LRU cache
    (16 entries): 24 steps on freshly allocated tensors (every step a new tuple, evictions
    from step 17 on) give bitwise the losses of the same 24 batches fed through one reused
    tuple (one graph)."""
    cfg = crl_synth.preset("reacher", batch=64, width=64, precision="bf16")
    ctx_a, _ = make_ctx(cfg)
    ctx_b, _ = make_ctx(cfg)
    sb, ab, gb = (torch.empty(64, cfg[k], device="cuda") for k in ("obs_dim", "act_dim", "goal_dim"))
    lb = torch.zeros(4, device="cuda")
    for it in range(24):
        s, a, g = (torch.from_numpy(x).cuda() for x in crl_synth.random_batch(cfg, 64, seed=500 + it))
        la = torch.zeros(4, device="cuda")
        ctx_a.critic_step(s, a, g, la)
        sb.copy_(s); ab.copy_(a); gb.copy_(g)
        ctx_b.critic_step(sb, ab, gb, lb)
        torch.cuda.synchronize()
        assert np.array_equal(la.cpu().numpy().view(np.uint32), lb.cpu().numpy().view(np.uint32)), it
    assert ctx_a.status() == 0 and ctx_b.status() == 0


@pytest.mark.parametrize("batch,width,repr_dim", [
    (300, 1024, 256),     # ragged last 256-row tile of the CTA-pair GEMM
    (1100, 320, 64),      # N = 320: a partial 256-column tile (one 64-column chunk)
    (640, 256, 256),      # width 256, D 256: one N tile per layer, output layer N = 256
])
def test_critic_step_bf16_pair_gemm_shapes(batch, width, repr_dim):
    """The persistent CTA-pair GEMM (tc_pgemm.cu: tcgen05 cta_group::2, 256 x 256 tiles, double
    TMEM accumulator) serves every forward / dX product with N >= 256; ragged M and N tiles."""
    cfg = crl_synth.preset("ant", batch=batch, width=width, repr_dim=repr_dim, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("energy", ["l2", "cos"])
@pytest.mark.parametrize("batch", [1100, 3000])
def test_critic_step_bf16_stats_d256(energy, batch):
    """The one-pass row + column statistics (tc_stats.cu) at D = 256 (configs[4]'s repr dim):
    the B tile staged in two 32 KB K pieces, a single A buffer per unit, ragged N."""
    cfg = crl_synth.preset("ant", batch=batch, width=256, repr_dim=256, energy=energy, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("energy,knob", [
    ("l2", None), ("dot", None), ("cos", None),
    ("l2", "CRL_FORCE_EXACT_Q"),      # exact second exp2 instead of the row / column factors
    ("cos", "CRL_FORCE_EXACT_Q"),
    ("l2", "CRL_NO_GRAD2P"),          # the single-CTA pass instead of the CTA-pair one
    ("cos", "CRL_NO_GRAD2P"),
    ("l2", "CRL_NO_GRAD2"),           # the two-call gradient kernels (tc_logits.cu)
    ("dot", "CRL_NO_GRAD2"),
])
@pytest.mark.parametrize("batch", [1100, 2900])
def test_critic_step_bf16_grad2_d256(energy, knob, batch, monkeypatch):
    """The both-sides gradient pass at D = 256 (tc_grad2.cu: persistent, contiguous tile ranges,
    A held in TMEM, two partial slots per cut row block; by default on CTA pairs, tc_grad2p)
    against the oracle; ragged N."""
    if knob:
        monkeypatch.setenv(knob, "1")
    cfg = crl_synth.preset("ant", batch=batch, width=256, repr_dim=256, energy=energy, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


def test_critic_step_bf16_wide_dw_long_k():
    """Weight / bias gradients of wide encoders with a long batch reduction (tc_dwg.cu: 2 K
    slices for width >= 512, 128 x 256 tiles, the bias sums by an all-ones MMA on M block 0)
    against the oracle, per tensor; a ragged batch (K not a multiple of the 64-row K block)
    and the 37-input first layer (one partial M block)."""
    cfg = crl_synth.preset("ant", batch=4160, width=512, repr_dim=64, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("preset,prec,batch,extra", [
    ("ant", "fp32", 300, {}),                       # SIMT logits with gathered Phi / Psi
    ("ant", "bf16", 1100, {}),                      # one-pass statistics + column-sum all-reduce (C2)
    ("ant", "bf16", 600, {"width": 256, "repr_dim": 256}),   # D = 256: tc_grad2p with gathered operands
])
def test_critic_step_forced_dist_path(preset, prec, batch, extra, monkeypatch):
    """The data-parallel schedule on one GPU: CRL_FORCE_DIST=1 runs world_size 1 through the
    multi-GPU code path -- a one-rank NCCL communicator, separate global gather buffers
    (Phi_g, Psi_g, LSE_g, factors), all-gathers, the loss all-reduce + finalize kernel, the
    split-partial reduction + gradient all-reduce before Adam -- against the oracle."""
    monkeypatch.setenv("CRL_FORCE_DIST", "1")
    cfg = crl_synth.preset(preset, precision=prec, batch=batch, **extra)
    tol = BF16_TOL if prec == "bf16" else None
    if tol is None:
        _critic_parity(cfg)
    else:
        _critic_parity(cfg, tol_loss=tol, tol_grad=tol)


@pytest.mark.parametrize("knobs", [
    {},                                        # defaults: pdw 256 x 512 items, merged pair GEMMs
    {"CRL_PDW_NH": "1"},                       # 256 x 256 dW items, double-buffered accumulators
    {"CRL_NO_PG_MERGE": "1"},                  # one pair-GEMM launch per encoder and layer
    {"CRL_PG_EPIW": "4"},                      # 4 epilogue warps on the short-K layers too
    {"CRL_PG_EPIW": "8"},                      # 8 epilogue warps on every layer
    {"CRL_NO_PDW": "1"},                       # the grouped single-CTA dW kernel
])
def test_critic_step_bf16_wide_kernel_variants(knobs, monkeypatch):
    """The wide-encoder kernels' selectable variants (round 2: tc_pdw items of 256 x 512 / 256 x
    256, tc_pgemm2 merged launches, 4 / 8 epilogue warps) against the oracle, per tensor: a
    ragged batch over 2 K slices and widths where the first / output layers are short-K."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    cfg = crl_synth.preset("ant", batch=1100, width=512, repr_dim=256, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("energy", ["l2", "l2sq", "dot"])
@pytest.mark.parametrize("loss,beta", [("sym", 0.0), ("fwd", 0.3), ("bwd", 0.0)])
@pytest.mark.parametrize("wsym", [True, False])
def test_critic_step_bf16_d256_stored_w(energy, loss, beta, wsym, monkeypatch):
    """D = 256 gradient at W = 1 for the symmetric energies: the pair pass computes side 0 only,
    stores W = dL/dS (bf16) and dPsi = W^T Phi plus the column sums of W come from one pair GEMM
    (tc_pdw.cu); CRL_NO_G2_WSYM keeps both sides in the pass.  Ragged batch (the last row-block
    pair half empty; one side's 45 tiles over 10 pairs cut row blocks into 3 partial slots), every
    loss kind, a logsumexp penalty.  Checked: the loss, both LSE vectors and the path's outputs
    dPhi / dPsi (norm and element-wise).  The encoder gradients behind them are not: at this
    random-init shape they are ill-conditioned in dPhi (the oracle alone, dPhi perturbed by 0.4 %
    element-wise noise, moves them by 2-3 %: above the bf16 bar for BOTH paths); the stored-W
    path's full gradient is checked at the 4 x 1024 shapes (test_critic_step_bf16_repr256_width1024)."""
    if not wsym:
        monkeypatch.setenv("CRL_NO_G2_WSYM", "1")
    cfg = crl_synth.preset("ant", batch=1100, width=128, repr_dim=256, energy=energy, loss=loss,
                           beta_lse=beta, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL, encoder_grads=False)


def test_critic_step_bf16_netscale_shapes_bitwise_deterministic():
    """Two fresh contexts, same parameters and batch, at the 4 x 1024 / D = 256 shapes: the loss,
    dPhi, dPsi and the whole pre-Adam gradient agree bit for bit -- the stored-W pass and its
    column GEMM (fixed K slices), the row-side merge on the second stream, the ticketed loss and
    the dW slices summed in a fixed order are deterministic (no float atomics on this path)."""
    cfg = crl_synth.preset("netscale", batch=1024)
    s, a, g = crl_synth.random_batch(cfg, 1024, seed=21)
    outs = []
    for _ in range(2):
        ctx, _p = make_ctx(cfg)
        loss = torch.zeros(4, device="cuda")
        grads = torch.zeros(ctx.n_params, device="cuda")
        ctx.critic_step(*(torch.from_numpy(x).cuda() for x in (s, a, g)), loss, grads)
        torch.cuda.synchronize()
        assert ctx.status() == 0
        outs.append([loss.cpu().numpy(), ctx.debug_tensor("dphi").cpu().numpy(),
                     ctx.debug_tensor("dpsi").cpu().numpy(), grads.cpu().numpy()])
        del ctx
    for x, y in zip(*outs):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("batch", [256, 300, 640])
def test_critic_step_bf16_d256_stored_w_small(batch, monkeypatch):
    """The stored-W path at its smallest batches: one row-block pair (256), a half-empty second
    pair whose rank-1 rows are all past the batch (300: its W stores are skipped, its columns
    clipped) and 2.5 pairs (640), each with the row-side merge on the second stream; outputs
    dPhi / dPsi and the loss against the oracle (encoder gradients: see stored_w above)."""
    cfg = crl_synth.preset("ant", batch=batch, width=128, repr_dim=256, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL, encoder_grads=False)


@pytest.mark.parametrize("energy", ["l2sq", "dot"])
def test_critic_step_bf16_width1024_stored_w_energies(energy):
    """The stored-W gradient path's full pre-Adam gradient (every W, b of both encoders) for the
    other symmetric energies at the configs[4] network shapes (well-conditioned: 0.4 % noise on
    dPhi moves the encoder gradients by < 0.4 % here)."""
    cfg = crl_synth.preset("netscale", batch=512, energy=energy)
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)


@pytest.mark.parametrize("buckets", ["1", "3", "8"])
def test_critic_step_forced_dist_buckets(buckets, monkeypatch):
    """C4: the gradient all-reduce in 1 / 3 / 8 buckets (bucket sizes rounded to 256 floats, a
    short last bucket, Adam per bucket on the communication-stream events) on the one-rank
    communicator, against the oracle."""
    monkeypatch.setenv("CRL_FORCE_DIST", "1")
    monkeypatch.setenv("CRL_AR_BUCKETS", buckets)
    cfg = crl_synth.preset("ant", batch=600, precision="bf16")
    _critic_parity(cfg, tol_loss=BF16_TOL, tol_grad=BF16_TOL)
