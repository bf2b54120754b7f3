"""GPU parity of crl_actor_loss (Eq. 3, entropy term P:313, readings A-26/A-27)
against oracle/critic.py actor_loss on the same seeded inputs.

Bar (north_star): the actor path is fp32 throughout (the frozen critic's fp32 master
weights), so loss within 1e-5 relative and gradients within 1e-4 relative; the Adam step is
checked against oracle Adam applied to the GPU gradients (1e-5), so only the update rule is
under test there."""
import numpy as np
import pytest

import crl_synth
from _crl_testlib import rel

pytestmark = pytest.mark.gpu


def _ctx(cfg, actor_params, world=1, rank=0):
    import torch
    from paper_2408_11052_b200 import CrlConfig, CrlContext
    c = CrlConfig.from_preset(cfg, world_size=world, rank=rank, actor_depth=2, actor_width=256)
    critic = crl_synth.init_critic_params(cfg, 42)
    ctx = CrlContext(c, params=torch.from_numpy(critic), actor_params=torch.from_numpy(actor_params))
    return ctx, critic


def _run(cfg, alpha, seed=5, clip_bias=False, steps=1):
    import torch
    from oracle import critic as oc
    from oracle import adam as oa
    A = cfg["act_dim"]
    actor = crl_synth.init_actor_params(cfg, 43)
    if clip_bias:
        # push some log-sigma outputs outside [-5, 2] (reading A-27: clipped, zero gradient)
        b_off = actor.size - 2 * A
        for k in range(A):
            actor[b_off + A + k] = 3.0 if k % 2 == 0 else -6.0
    ctx, critic = _ctx(cfg, actor)
    N = cfg["batch"]
    s, _, g = crl_synth.random_batch(cfg, N, seed=seed)
    eps = np.random.default_rng(seed + 100).standard_normal((N, A)).astype(np.float32)
    ds, dg, de = (torch.from_numpy(x).cuda() for x in (s, g, eps))
    loss = torch.zeros(1, device="cuda")
    grads = torch.zeros(ctx.sizes["n_actor_params"], device="cuda")
    p_host = actor.astype(np.float64)
    m = np.zeros_like(p_host); v = np.zeros_like(p_host); t = 0
    for it in range(steps):
        ctx.actor_loss(ds, dg, de, alpha, loss_out=loss, actor_grads_out=grads, apply_adam=True)
        torch.cuda.synchronize()
        assert ctx.status() == 0
        ref = oc.actor_loss(p_host, critic, s, g, eps, alpha_ent=alpha, obs_dim=cfg["obs_dim"],
                            act_dim=A, goal_dim=cfg["goal_dim"], depth=cfg["depth"], width=cfg["width"],
                            repr_dim=cfg["repr_dim"], actor_depth=2, actor_width=256,
                            energy_kind=cfg["energy"], activation=cfg["activation"])
        gl = float(loss.cpu()[0])
        gg = grads.cpu().numpy().astype(np.float64)
        assert abs(gl - ref["loss"]) <= 1e-5 * max(abs(ref["loss"]), 1e-3), (it, gl, ref["loss"])
        assert rel(gg, ref["grads"]) < 1e-4, (it, rel(gg, ref["grads"]))
        # Adam on the GPU's gradients (lr_actor, Table 2)
        p_host, m, v, t = oa.adam_step(p_host, gg, m, v, t, lr=ctx.cfg.lr_actor, b1=ctx.cfg.adam_b1,
                                       b2=ctx.cfg.adam_b2, eps=ctx.cfg.adam_eps, wd=ctx.cfg.weight_decay)
        gp = ctx.actor_params.cpu().numpy().astype(np.float64)
        assert rel(gp - actor, p_host - actor) < 1e-4, rel(gp - actor, p_host - actor)
        p_host = gp                       # continue from the GPU's parameters
    return ref


@pytest.mark.parametrize("preset,energy,act,alpha", [
    ("reacher", "l2", "silu", 0.1),
    ("ant", "dot", "silu", 0.0),         # alpha = 0: random-goal setting (App. C)
    ("ant", "cos", "relu", 0.05),
    ("humanoid", "l2", "silu", 0.1),     # obs 268, act 17 (wide first layers, ragged tiles)
    ("reacher", "l1", "silu", 0.1),      # F3 energies
    ("ant", "l2sq", "relu", 0.05),
])
def test_actor_loss_parity(preset, energy, act, alpha):
    cfg = crl_synth.preset(preset, energy=energy, activation=act)
    _run(cfg, alpha)


def test_actor_loss_log_sigma_clip():
    cfg = crl_synth.preset("reacher", batch=200)   # ragged batch
    _run(cfg, 0.2, clip_bias=True)


def test_actor_loss_two_steps():
    cfg = crl_synth.preset("ant", batch=128)
    _run(cfg, 0.1, steps=2)


def test_actor_loss_without_actor_is_unsupported():
    import torch
    from paper_2408_11052_b200 import CrlConfig, CrlContext, CrlError
    cfg = crl_synth.preset("reacher")
    c = CrlConfig.from_preset(cfg)
    ctx = CrlContext(c, params=torch.from_numpy(crl_synth.init_critic_params(cfg)))
    z = torch.zeros(cfg["batch"], 16, device="cuda")
    with pytest.raises(CrlError) as e:
        ctx.actor_loss(z, z, z, 0.1)
    assert e.value.code == 7             # CRL_EUNSUPPORTED


def test_entropy_update_parity():
    """crl_entropy_update (reading A-32) against oracle/critic.py entropy_update over three
    Adam steps, fed the oracle's log pi of the same actor call (the GPU's mean log pi is fp32:
    1e-5 relative on the loss, 1e-6 absolute on log alpha)."""
    import torch
    from oracle import critic as oc
    cfg = crl_synth.preset("ant", batch=300)
    A = cfg["act_dim"]
    actor = crl_synth.init_actor_params(cfg, 43)
    ctx, critic = _ctx(cfg, actor)
    N = cfg["batch"]
    s, _, g = crl_synth.random_batch(cfg, N, seed=9)
    eps = np.random.default_rng(109).standard_normal((N, A)).astype(np.float32)
    ds, dg, de = (torch.from_numpy(x).cuda() for x in (s, g, eps))
    log_alpha = torch.full((1,), np.log(0.1), dtype=torch.float32, device="cuda")
    alpha = torch.zeros(1, device="cuda")
    lossa = torch.zeros(1, device="cuda")
    from paper_2408_11052_b200 import CrlError
    with pytest.raises(CrlError):                  # no actor loss yet: CRL_ESTATE
        ctx.entropy_update(log_alpha, lr=1e-2)
    ctx.actor_loss(ds, dg, de, 0.1)
    ref = oc.actor_loss(actor.astype(np.float64), critic, s, g, eps, alpha_ent=0.1, obs_dim=cfg["obs_dim"],
                        act_dim=A, goal_dim=cfg["goal_dim"], depth=cfg["depth"], width=cfg["width"],
                        repr_dim=cfg["repr_dim"], actor_depth=2, actor_width=256,
                        energy_kind=cfg["energy"], activation=cfg["activation"])
    H = -0.5 * A
    la, m, v, t = float(np.float32(np.log(0.1))), 0.0, 0.0, 0
    for it in range(3):
        ctx.entropy_update(log_alpha, target_entropy=H, lr=1e-2, alpha_out=alpha, loss_out=lossa)
        torch.cuda.synchronize()
        assert ctx.status() == 0
        o = oc.entropy_update(ref["log_pi"], la, m, v, t, target_entropy=H, lr=1e-2, b1=ctx.cfg.adam_b1,
                              b2=ctx.cfg.adam_b2, eps=ctx.cfg.adam_eps)
        assert abs(float(lossa.cpu()[0]) - o["loss"]) <= 1e-5 * abs(o["loss"]), (it, float(lossa.cpu()[0]), o)
        assert abs(float(log_alpha.cpu()[0]) - o["log_alpha"]) <= 1e-6, (it, float(log_alpha.cpu()[0]), o)
        assert abs(float(alpha.cpu()[0]) - o["alpha"]) <= 1e-6 * o["alpha"] + 1e-7
        la, m, v, t = o["log_alpha"], o["m"], o["v"], o["t"]
