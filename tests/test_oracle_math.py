"""Pins for oracle/mlp.py, energy.py, losses.py, adam.py, critic.py (contracts C2-C8), CPU.

Every pin is independent of the function it checks: hand values and closed forms from the
paper's definitions (tests/golden/closed_forms.txt), invariants (shift invariance, row /
column sums of the softmax gradient, sign and range of the energies), and central finite
differences in fp64 of the scalar loss through the whole path."""
import math

import numpy as np
import pytest

from oracle import adam, critic, energy, losses, mlp

ENERGIES = ["l2", "dot", "cos", "l1", "l2sq"]
KINDS = ["fwd", "bwd", "sym"]


def fd_grad(f, x, h=1e-6):
    x = np.array(x, np.float64)
    g = np.zeros_like(x)
    flat, gf = x.ravel(), g.ravel()
    for i in range(flat.size):
        old = flat[i]
        flat[i] = old + h; fp = f(x)
        flat[i] = old - h; fm = f(x)
        flat[i] = old
        gf[i] = (fp - fm) / (2 * h)
    return g


def rel_err(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-30)


# ------------------------------------------------------------------------------ energies

def test_energy_hand_values(closed_forms):
    z, p = np.array([[0.0, 0.0]]), np.array([[3.0, 4.0]])
    assert abs(energy.logits("l2", z, p)[0, 0] - closed_forms["l2_345"]) < 1e-12
    assert energy.logits("dot", np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]))[0, 0] == closed_forms["dot_12_34"]
    u = np.array([[0.3, -1.2, 2.0]])
    assert abs(energy.logits("cos", u, u)[0, 0] - closed_forms["cos_identical"]) < 1e-15
    assert abs(energy.logits("cos", np.array([[1.0, 0]]), np.array([[0, 2.0]]))[0, 0]
               - closed_forms["cos_orthogonal"]) < 1e-15


def test_energy_ranges_and_diag():
    rng = np.random.default_rng(0)
    phi, psi = rng.standard_normal((9, 5)), rng.standard_normal((9, 5))
    l2 = energy.logits("l2", phi, psi)
    assert np.all(l2 < 0)
    assert abs(energy.logits("l2", phi, phi)[3, 3] + 1e-6) < 1e-12       # -sqrt(eps2)
    c = energy.logits("cos", phi, psi)
    assert np.all(np.abs(c) <= 1 + 1e-12)
    for k in ENERGIES:
        assert np.allclose(np.diag(energy.logits(k, phi, psi)), energy.diag_logits(k, phi, psi))
    # L2 logits are symmetric in their two arguments
    assert np.allclose(energy.logits("l2", phi, psi), energy.logits("l2", psi, phi).T)


@pytest.mark.parametrize("kind", ENERGIES)
def test_energy_vjp_finite_differences(kind):
    rng = np.random.default_rng(1)
    N, D = 5, 4
    phi, psi = rng.standard_normal((N, D)), rng.standard_normal((N, D))
    G = rng.standard_normal((N, N))
    dphi, dpsi = energy.vjp(kind, phi, psi, G)
    fphi = fd_grad(lambda x: (energy.logits(kind, x, psi) * G).sum(), phi)
    fpsi = fd_grad(lambda x: (energy.logits(kind, phi, x) * G).sum(), psi)
    assert rel_err(dphi, fphi) < 1e-7
    assert rel_err(dpsi, fpsi) < 1e-7


# ------------------------------------------------------------------------------ losses

def test_loss_closed_forms(closed_forms):
    z = np.zeros((2, 2))
    c, _ = losses.loss_and_grad(z, "fwd", 0.1)
    assert abs(c["L_fwd"] - closed_forms["infonce_fwd_zero2x2"]) < 1e-15
    assert abs(c["penalty"] - closed_forms["penalty_zero2x2_b01"]) < 1e-15
    c, _ = losses.loss_and_grad(z, "sym", 0.0)
    assert abs(c["total"] - closed_forms["infonce_sym_zero2x2"]) < 1e-15
    c, _ = losses.loss_and_grad(np.eye(2), "fwd", 0.0)
    assert abs(c["total"] - closed_forms["infonce_fwd_eye2"]) < 1e-15
    I4 = np.eye(4)
    c, _ = losses.loss_and_grad(energy.logits("dot", I4, I4), "fwd", 0.0)
    assert abs(c["total"] - closed_forms["infonce_fwd_onehot4"]) < 1e-14
    c, _ = losses.loss_and_grad(energy.logits("l2", I4, I4), "fwd", 0.0)
    assert abs(c["total"] - closed_forms["infonce_fwd_orthl2_4"]) < 1e-5   # eps2 = 1e-12 perturbs


@pytest.mark.parametrize("N", [3, 8])
def test_loss_all_equal_logits(N):
    cval, beta = -2.5, 0.1
    comps, _ = losses.loss_and_grad(np.full((N, N), cval), "sym", beta)
    assert abs(comps["L_fwd"] - math.log(N)) < 1e-13
    assert abs(comps["L_bwd"] - math.log(N)) < 1e-13
    assert abs(comps["penalty"] - beta * (cval + math.log(N)) ** 2) < 1e-13


def test_loss_shift_invariance_and_gradient_sums():
    rng = np.random.default_rng(2)
    l = rng.standard_normal((6, 6))
    a, _ = losses.loss_and_grad(l, "sym", 0.1)
    b, _ = losses.loss_and_grad(l + 3.7, "sym", 0.1)
    assert abs(a["L_fwd"] - b["L_fwd"]) < 1e-13 and abs(a["L_bwd"] - b["L_bwd"]) < 1e-13
    assert abs(a["penalty"] - b["penalty"]) > 1e-3                     # penalty is not invariant
    assert np.allclose(b["lse_row"], a["lse_row"] + 3.7)
    _, Gf = losses.loss_and_grad(l, "fwd", 0.0)
    _, Gb = losses.loss_and_grad(l, "bwd", 0.0)
    assert np.allclose(Gf.sum(1), 0, atol=1e-15)                        # softmax rows sum to 1
    assert np.allclose(Gb.sum(0), 0, atol=1e-15)
    _, Gs = losses.loss_and_grad(l, "sym", 0.0)
    assert np.allclose(Gs, Gf + Gb, rtol=0, atol=1e-16)
    cs, _ = losses.loss_and_grad(l, "sym", 0.0)
    cf, _ = losses.loss_and_grad(l, "fwd", 0.0)
    cb, _ = losses.loss_and_grad(l, "bwd", 0.0)
    assert cs["total"] == cf["total"] + cb["total"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("beta", [0.0, 0.1])
def test_loss_gradient_finite_differences(kind, beta):
    rng = np.random.default_rng(3)
    l = rng.standard_normal((5, 5)) * 2
    _, G = losses.loss_and_grad(l, kind, beta)
    fd = fd_grad(lambda x: losses.loss_and_grad(x, kind, beta)[0]["total"], l)
    assert rel_err(G, fd) < 1e-8


def test_loss_increasing_diagonal_lowers_loss():
    rng = np.random.default_rng(4)
    l = rng.standard_normal((7, 7))
    for k in KINDS:
        a, _ = losses.loss_and_grad(l, k, 0.0)
        b, _ = losses.loss_and_grad(l + 0.5 * np.eye(7), k, 0.0)
        assert b["total"] < a["total"]


# ------------------------------------------------------------------------------ MLP

def test_mlp_zero_weights_gives_output_bias():
    rng = np.random.default_rng(5)
    dims = mlp.layer_dims(4, 2, 6, 3)
    layers = [(np.zeros(d), rng.standard_normal(d[1]) if i == len(dims) - 1 else rng.standard_normal(d[1]))
              for i, d in enumerate(dims)]
    layers = [(np.zeros((fi, fo)), b) for (fi, fo), (_, b) in zip(dims, layers)]
    y, _ = mlp.forward(layers, rng.standard_normal((5, 4)), "silu")
    assert np.allclose(y, layers[-1][1][None, :])


def test_mlp_linear_layer_closed_form():
    rng = np.random.default_rng(6)
    W, b = rng.standard_normal((4, 3)), rng.standard_normal(3)
    X, dY = rng.standard_normal((6, 4)), rng.standard_normal((6, 3))
    y, cache = mlp.forward([(W, b)], X)
    assert np.allclose(y, X @ W + b)
    (gw, gb), = mlp.backward([(W, b)], cache, dY)[0]
    assert np.allclose(gw, sum(np.outer(X[i], dY[i]) for i in range(6)))
    assert np.allclose(gb, dY.sum(0))


@pytest.mark.parametrize("act", ["silu", "relu"])
def test_mlp_backward_finite_differences(act):
    rng = np.random.default_rng(7)
    layers = [(rng.standard_normal((fi, fo)) * 0.7, rng.standard_normal(fo) * 0.3)
              for fi, fo in mlp.layer_dims(3, 2, 5, 4)]
    X, C = rng.standard_normal((6, 3)), rng.standard_normal((6, 4))
    flat = mlp.pack(layers)

    def f(p):
        ls, _ = mlp.unpack(p, 3, 2, 5, 4)
        return (mlp.forward(ls, X, act)[0] * C).sum()

    _, cache = mlp.forward(layers, X, act)
    grads, _ = mlp.backward(layers, cache, C, act)
    assert rel_err(mlp.pack(grads), fd_grad(f, flat)) < 1e-7


def test_activation_values():
    z = np.array([-2.0, 0.0, 1.5])
    assert np.allclose(mlp.act_fn(z, "silu"), z / (1 + np.exp(-z)))
    assert mlp.act_fn(np.array([0.0]), "silu")[0] == 0.0
    assert mlp.act_grad(np.array([0.0]), "relu")[0] == 0.0
    assert abs(mlp.act_grad(np.array([0.0]), "silu")[0] - 0.5) < 1e-15


# ------------------------------------------------------------------------------ Adam

def test_adam_zero_gradient_is_identity():
    p = np.array([1.0, -2.0, 3.0])
    p2, m2, v2, t2 = adam.adam_step(p, np.zeros(3), np.zeros(3), np.zeros(3), 0)
    assert np.array_equal(p2, p) and t2 == 1


def test_adam_first_step_closed_form():
    g = np.array([1e-3, -2.0, 5e-9, 0.3])
    p2, *_ = adam.adam_step(np.zeros(4), g, np.zeros(4), np.zeros(4), 0, lr=0.01)
    assert np.allclose(p2, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)


def test_adam_quadratic_recurrence():
    th, m, v, t = np.array([1.0]), np.zeros(1), np.zeros(1), 0
    for _ in range(100):
        th, m, v, t = adam.adam_step(th, 2 * th, m, v, t, lr=0.1)
    assert abs(th[0]) < 0.1


def test_adam_rejects_non_finite():
    with pytest.raises(FloatingPointError):
        adam.adam_step(np.zeros(2), np.array([np.nan, 0]), np.zeros(2), np.zeros(2), 0)


# ------------------------------------------------------------------------------ whole step

TINY = dict(obs_dim=3, act_dim=2, goal_dim=2, depth=2, width=5, repr_dim=4)


def _tiny_problem(seed, N=6):
    rng = np.random.default_rng(seed)
    n_phi = sum(i * o + o for i, o in mlp.layer_dims(5, 2, 5, 4))
    n_psi = sum(i * o + o for i, o in mlp.layer_dims(2, 2, 5, 4))
    params = rng.standard_normal(n_phi + n_psi) * 0.6
    s, a, g = rng.standard_normal((N, 3)), rng.uniform(-1, 1, (N, 2)), rng.standard_normal((N, 2))
    return params, s, a, g


@pytest.mark.parametrize("kind", ENERGIES)
@pytest.mark.parametrize("loss_kind", KINDS)
@pytest.mark.parametrize("act", ["silu", "relu"])
def test_critic_gradient_end_to_end_finite_differences(kind, loss_kind, act):
    params, s, a, g = _tiny_problem(8)
    kw = dict(TINY, energy_kind=kind, loss_kind=loss_kind, beta=0.1, activation=act)
    out = critic.critic_forward_backward(params, s, a, g, **kw)
    fd = fd_grad(lambda p: critic.critic_forward_backward(p, s, a, g, **kw)["total"], params)
    assert rel_err(out["grads"], fd) < 1e-6


def test_critic_step_applies_adam_to_the_gradient():
    params, s, a, g = _tiny_problem(9)
    z = np.zeros_like(params)
    out = critic.critic_step(params, z, z, 0, s, a, g, lr=1e-3, **TINY)
    gr = out["grads"]
    assert np.allclose(out["params_new"], params - 1e-3 * gr / (np.abs(gr) + 1e-8))
    assert out["t_new"] == 1


def test_critic_step_descends():
    params, s, a, g = _tiny_problem(10, N=8)
    p, m, v, t = params, np.zeros_like(params), np.zeros_like(params), 0
    l0 = critic.critic_forward_backward(p, s, a, g, **TINY)["total"]
    for _ in range(5):
        o = critic.critic_step(p, m, v, t, s, a, g, lr=1e-2, **TINY)
        p, m, v, t = o["params_new"], o["m_new"], o["v_new"], o["t_new"]
    assert critic.critic_forward_backward(p, s, a, g, **TINY)["total"] < l0


@pytest.mark.parametrize("kind", ENERGIES)
def test_actor_loss_finite_differences(kind):
    rng = np.random.default_rng(11)
    N = 5
    params, s, _, g = _tiny_problem(12, N=N)
    n_pi = sum(i * o + o for i, o in mlp.layer_dims(5, 2, 6, 4))
    pi = rng.standard_normal(n_pi) * 0.5
    eps = rng.standard_normal((N, 2))
    kw = dict(TINY, actor_depth=2, actor_width=6, energy_kind=kind, alpha_ent=0.2)
    out = critic.actor_loss(pi, params, s, g, eps, **kw)
    fd = fd_grad(lambda p: critic.actor_loss(p, params, s, g, eps, **kw)["loss"], pi)
    assert rel_err(out["grads"], fd) < 1e-6
    assert np.all(np.abs(out["a_new"]) < 1)


def test_bf16_round_is_round_to_nearest_even():
    x = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, -3.14159], np.float32)
    r = critic.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0 + 2**-6 and abs(r[3] + 3.140625) < 1e-12


# ------------------------------------------------------------------ entropy coefficient (A-32)

def test_entropy_update_first_step_closed_form():
    """First Adam step from zero moments: m^ = g, v^ = g^2, so log_alpha moves by exactly
    -lr g / (|g| + eps); g = alpha (-mean log pi - H)."""
    log_pi = np.array([-1.5, -0.5, -2.0, -1.0])            # mean -1.25
    la, H, lr = math.log(0.2), -2.0, 1e-3
    out = critic.entropy_update(log_pi, la, 0.0, 0.0, 0, target_entropy=H, lr=lr)
    g = 0.2 * (1.25 - (-2.0))                               # alpha (-mean - H) = 0.2 * 3.25
    assert out["loss"] == pytest.approx(g, rel=1e-15)
    assert out["log_alpha"] == pytest.approx(la - lr * g / (abs(g) + 1e-8), rel=1e-15)
    assert out["alpha"] == pytest.approx(math.exp(out["log_alpha"]), rel=1e-15)
    assert out["t"] == 1


def test_entropy_update_direction():
    """Policy entropy above the target (-mean log pi > H) lowers alpha; below raises it."""
    H = -3.0
    hi = critic.entropy_update(np.full(8, 1.0), 0.0, 0.0, 0.0, 0, target_entropy=H, lr=1e-2)
    lo = critic.entropy_update(np.full(8, 5.0), 0.0, 0.0, 0.0, 0, target_entropy=H, lr=1e-2)
    assert hi["alpha"] < 1.0 < lo["alpha"]


def test_entropy_update_gradient_finite_difference():
    """The Adam input is dL/dlog_alpha: check it against a central difference of
    L(log_alpha) = exp(log_alpha) (-mean log pi - H) (zero-lr call exposes the loss)."""
    log_pi = np.array([0.3, -0.7, 1.1])
    H, la, h = 0.5, -0.4, 1e-6
    f = lambda x: critic.entropy_update(log_pi, x, 0, 0, 0, target_entropy=H, lr=1e-30)["loss"]
    fd = (f(la + h) - f(la - h)) / (2 * h)
    assert f(la) == pytest.approx(fd, rel=1e-8)


# ------------------------------------------------------------------ F3 energies (L1, L2 w/o sqrt)

def test_l2sq_and_l1_logits_closed_forms():
    """App. A.2 P:612/P:616 on integer vectors: -||x - y||_2^2 and -||x - y||_1 by hand."""
    phi = np.array([[1.0, 2.0, -1.0], [0.0, 0.0, 0.0]])
    psi = np.array([[0.0, 4.0, 1.0], [1.0, 1.0, 1.0], [-2.0, 2.0, 0.5]])
    l2sq = energy.logits("l2sq", phi, psi)
    l1 = energy.logits("l1", phi, psi)
    assert l2sq[0, 0] == -(1 + 4 + 4) and l2sq[1, 1] == -3 and l2sq[0, 2] == -(9 + 0 + 2.25)
    assert l1[0, 0] == -(1 + 2 + 2) and l1[1, 1] == -3 and l1[0, 2] == -(3 + 0 + 1.5)
    # L2sq is the square of the L2 distance (up to the L2 epsilon)
    l2 = energy.logits("l2", phi, psi)
    assert np.allclose(-l2sq, l2 ** 2 - energy.EPS_L2, rtol=1e-12, atol=1e-12)
    assert np.allclose(energy.diag_logits("l1", phi, psi[:2]), np.diag(l1[:, :2]))
    assert np.allclose(energy.diag_logits("l2sq", phi, psi[:2]), np.diag(l2sq[:, :2]))


@pytest.mark.parametrize("kind", ["l1", "l2sq"])
def test_l1_l2sq_vjp_finite_differences(kind):
    """The VJPs of the F3 energies against central differences of sum(G * logits) (random
    points: no L1 ties within the step)."""
    rng = np.random.default_rng(3)
    phi = rng.standard_normal((5, 4)); psi = rng.standard_normal((6, 4)); G = rng.standard_normal((5, 6))
    dphi, dpsi = energy.vjp(kind, phi, psi, G)
    f = lambda P, Q: float((G * energy.logits(kind, P, Q)).sum())
    h = 1e-6
    for (i, k) in [(0, 0), (2, 3), (4, 1)]:
        e = np.zeros_like(phi); e[i, k] = h
        assert (f(phi + e, psi) - f(phi - e, psi)) / (2 * h) == pytest.approx(dphi[i, k], rel=1e-6, abs=1e-8)
    for (j, k) in [(0, 1), (5, 2), (3, 0)]:
        e = np.zeros_like(psi); e[j, k] = h
        assert (f(phi, psi + e) - f(phi, psi - e)) / (2 * h) == pytest.approx(dpsi[j, k], rel=1e-6, abs=1e-8)


def test_l1_subgradient_at_ties_is_zero():
    """Reading A-33: at phi_k == psi_k the L1 derivative is taken as 0."""
    phi = np.array([[1.0, 2.0]]); psi = np.array([[1.0, 0.0]])
    dphi, dpsi = energy.vjp("l1", phi, psi, np.ones((1, 1)))
    assert dphi[0, 0] == 0.0 and dpsi[0, 0] == 0.0
    assert dphi[0, 1] == -1.0 and dpsi[0, 1] == 1.0


# ------------------------------------------------------------------ F3 FlatNCE (reading A-24)

@pytest.mark.parametrize("kind", ["flatnce_fwd", "flatnce_bwd"])
def test_flatnce_value_zero_and_gradient_of_literal_formula(kind):
    """The printed FlatNCE objective with the stop-gradient held at the evaluation point: its
    value there is 0 and its finite-difference gradient equals the oracle's G (independent of
    the InfoNCE closed form it coincides with)."""
    rng = np.random.default_rng(21)
    l = rng.standard_normal((5, 5))
    comps, G = losses.loss_and_grad(l, kind, beta=0.0)
    assert comps["L_fwd"] == 0.0 and comps["L_bwd"] == 0.0 and comps["total"] == 0.0
    assert losses.flatnce_literal(l, l, kind) == 0.0
    fd = fd_grad(lambda x: losses.flatnce_literal(x, l, kind), l)
    assert rel_err(G, fd) < 1e-7
    # and it is the InfoNCE gradient of the same direction
    _, Gi = losses.loss_and_grad(l, "fwd" if kind == "flatnce_fwd" else "bwd", beta=0.0)
    assert np.allclose(G, Gi, rtol=0, atol=1e-15)


def test_flatnce_penalty_only_total():
    l = np.random.default_rng(2).standard_normal((4, 4))
    c, _ = losses.loss_and_grad(l, "flatnce_fwd", beta=0.1)
    assert c["total"] == c["penalty"] > 0.0


# ------------------------------------------------------------------ F3 pairwise / FB losses

@pytest.mark.parametrize("N", [2, 5])
def test_pairwise_losses_closed_forms_at_zero_logits(N):
    """l = 0: DPO = N log 2 (N^2 terms log 2, mean over N), IPO = N, SPPO = 2 N, FB = -1/2."""
    z = np.zeros((N, N))
    assert losses.pairwise_loss(z, "dpo") == pytest.approx(N * math.log(2.0), rel=1e-15)
    assert losses.pairwise_loss(z, "ipo") == pytest.approx(N, rel=1e-15)
    assert losses.pairwise_loss(z, "sppo") == pytest.approx(2 * N, rel=1e-15)
    assert losses.pairwise_loss(z, "fb") == pytest.approx(-0.5, rel=1e-15)


@pytest.mark.parametrize("kind", ["fb", "dpo", "ipo", "sppo"])
@pytest.mark.parametrize("beta", [0.0, 0.1])
def test_pairwise_gradient_finite_differences(kind, beta):
    rng = np.random.default_rng(7)
    l = rng.standard_normal((6, 6)) * 0.7
    comps, G = losses.loss_and_grad(l, kind, beta)
    fd = fd_grad(lambda x: losses.loss_and_grad(x, kind, beta)[0]["total"], l)
    assert rel_err(G, fd) < 1e-7
    assert comps["total"] == pytest.approx(comps["L_fwd"] + comps["penalty"], rel=1e-15)


def test_ipo_sppo_minimisers():
    """IPO is zero exactly when every positive beats every negative by 1 (and the j = i term
    contributes (0 - 1)^2 = 1 per row); SPPO's off-diagonal part vanishes at l_ij = -1."""
    N = 4
    l = -np.ones((N, N)); np.fill_diagonal(l, 0.0)
    assert losses.pairwise_loss(l, "ipo") == pytest.approx(1.0, rel=1e-15)   # (1/N) * N rows * 1
    l2 = -np.ones((N, N)); np.fill_diagonal(l2, 1.0)
    # SPPO: diag (d-1)^2 = 0; (l+1)^2 = 0 off-diagonal, (1+1)^2 = 4 on the diagonal: (1/N) N 4
    assert losses.pairwise_loss(l2, "sppo") == pytest.approx(4.0, rel=1e-15)


# ------------------------------------------------------------------ F2 LayerNorm encoders (A-35)

def _ln_params(rng, in_dim, depth, width, out_dim):
    parts = []
    for li, (fi, fo) in enumerate(mlp.layer_dims(in_dim, depth, width, out_dim)):
        parts += [rng.standard_normal(fi * fo) / np.sqrt(fi), rng.standard_normal(fo) * 0.1]
        if li < depth:
            parts += [1.0 + 0.2 * rng.standard_normal(fo), 0.1 * rng.standard_normal(fo)]
    return np.concatenate(parts)


def test_layernorm_forward_properties():
    """With gamma = 1, beta = 0 every hidden pre-activation row has mean 0 and variance
    var / (var + eps) (~1); LN is invariant to a per-row shift and positive scale of Z."""
    rng = np.random.default_rng(4)
    p = _ln_params(rng, 5, 2, 16, 3)
    layers, n = mlp.unpack_ln(p, 5, 2, 16, 3)
    assert n == p.size
    layers = [(L[0], L[1], np.ones_like(L[2]), np.zeros_like(L[3])) if len(L) == 4 else L for L in layers]
    x = rng.standard_normal((7, 5))
    _, (Xs, Zs, Zhs, Ys, rs) = mlp.forward_ln(layers, x)
    for Y, Z in zip(Ys, Zs):
        assert np.allclose(Y.mean(1), 0.0, atol=1e-12)
        var = Z.var(1)
        assert np.allclose((Y ** 2).mean(1), var / (var + mlp.LN_EPS), rtol=1e-12)
    W0, b0, g0, bt0 = layers[0]
    lay2 = [(3.0 * W0, 3.0 * b0 + 0.0, g0, bt0)] + layers[1:]          # Z -> 3 Z: LN output unchanged (eps aside)
    y1, _ = mlp.forward_ln(layers, x); y2, _ = mlp.forward_ln(lay2, x)
    assert np.allclose(y1, y2, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("act", ["silu", "relu"])
def test_layernorm_mlp_gradient_finite_differences(act):
    rng = np.random.default_rng(5)
    p = _ln_params(rng, 4, 2, 8, 3)
    x = rng.standard_normal((6, 4))
    G = rng.standard_normal((6, 3))
    def f(q):
        L, _ = mlp.unpack_ln(q, 4, 2, 8, 3)
        return float((mlp.forward_ln(L, x, act)[0] * G).sum())
    L, _ = mlp.unpack_ln(p, 4, 2, 8, 3)
    _, cache = mlp.forward_ln(L, x, act)
    grads, _ = mlp.backward_ln(L, cache, G, act)
    assert rel_err(mlp.pack_ln(grads), fd_grad(f, p)) < 1e-7


def test_critic_layernorm_end_to_end_finite_differences():
    rng = np.random.default_rng(6)
    kw = dict(obs_dim=3, act_dim=2, goal_dim=2, depth=2, width=8, repr_dim=4, energy_kind="l2",
              loss_kind="sym", beta=0.1, activation="silu", layernorm=True)
    p = np.concatenate([_ln_params(rng, 5, 2, 8, 4), _ln_params(rng, 2, 2, 8, 4)])
    s, a, g = rng.standard_normal((6, 3)), rng.standard_normal((6, 2)), rng.standard_normal((6, 2))
    out = critic.critic_forward_backward(p, s, a, g, **kw)
    fd = fd_grad(lambda q: critic.critic_forward_backward(q, s, a, g, **kw)["total"], p)
    assert rel_err(out["grads"], fd) < 1e-6


# ------------------------------------------------------------------ policy log-density pins
# oracle/critic.py tanh_gaussian_sample_log_prob (Eq. 3: a' ~ pi(.|s, g); the
# tanh-squashed Gaussian and its change of variables, reading A-27).  Pinned against things
# other than its own formula: a closed form, scipy's normal log-density (the Gaussian part)
# and the normalisation of the density over the action box (the Jacobian part).

def test_log_pi_closed_form_at_the_origin():
    """mu = 0, log sigma = 0, eps = 0: u = 0, a' = 0, so
    log pi = -(k/2) log(2 pi) - k log(1 + 1e-6)."""
    for k in (1, 3, 17):
        a, lp = critic.tanh_gaussian_sample_log_prob(np.zeros((2, k)), np.zeros((2, k)), np.zeros((2, k)))
        assert np.all(a == 0.0)
        expect = -0.5 * k * np.log(2 * np.pi) - k * np.log(1.0 + 1e-6)
        assert np.allclose(lp, expect, rtol=0, atol=1e-13)


def test_log_pi_gaussian_part_matches_scipy():
    """log pi + sum_k log(1 - a'^2 + 1e-6) is the Gaussian log-density of u = mu + sigma eps:
    scipy.stats.norm.logpdf(u, mu, sigma) summed over the action dims."""
    from scipy.stats import norm
    rng = np.random.default_rng(3)
    mu = rng.normal(0, 0.7, (6, 4)); ls = rng.uniform(-2, 1, (6, 4)); eps = rng.standard_normal((6, 4))
    a, lp = critic.tanh_gaussian_sample_log_prob(mu, ls, eps)
    u = mu + np.exp(ls) * eps
    assert np.allclose(np.tanh(u), a, rtol=0, atol=1e-15)
    gauss = lp + np.log(1.0 - a ** 2 + 1e-6).sum(1)
    assert np.allclose(gauss, norm.logpdf(u, mu, np.exp(ls)).sum(1), rtol=0, atol=1e-12)


@pytest.mark.parametrize("mu,log_sig", [(0.0, 0.0), (0.3, -0.4), (-1.0, 0.5), (0.8, -2.0)])
def test_log_pi_density_integrates_to_one_over_the_action_box(mu, log_sig):
    """exp(log pi(a')) is a probability density on a' in (-1, 1): integrated by quadrature in
    u = atanh(a') (da' = (1 - tanh(u)^2) du) it gives 1 up to the 1e-6 guard, which removes
    E[1e-6 / (sech^2 u + 1e-6)] < 1e-3 of mass here (computed independently below).  A wrong sign of the Jacobian term, of
    log sigma or of the log(2 pi)/2 constant moves the integral by O(1)."""
    sig = np.exp(log_sig)
    u = np.linspace(mu - 12 * sig, mu + 12 * sig, 200001)
    eps = ((u - mu) / sig)[:, None]
    a, lp = critic.tanh_gaussian_sample_log_prob(np.full_like(eps, mu), np.full_like(eps, log_sig), eps)
    dens_a = np.exp(lp)                                   # density w.r.t. a'
    integrand = dens_a * (1.0 - np.tanh(u) ** 2)          # da' = sech^2(u) du
    total = np.trapezoid(integrand, u)
    # the mass the guard removes, from scipy's normal density (no oracle code):
    # int N(u; mu, sigma) sech^2(u) / (sech^2(u) + 1e-6) du
    from scipy.stats import norm
    sech2 = 1.0 / np.cosh(u) ** 2
    expect = np.trapezoid(norm.pdf(u, mu, sig) * sech2 / (sech2 + 1e-6), u)
    assert 1.0 - 1e-3 < expect <= 1.0
    assert abs(total - expect) < 1e-9, (total, expect)
