"""One CRL critic update and the CRL actor loss — oracle, fp64 (contracts C7, C8).

Critic (Alg. 1, §3.1):
  phi = phi_enc([s || a]),  psi = psi_enc(g)
  l_ij = f(phi_i, psi_j)                                         (App. A.2)
  L = L_critic(l) + beta L_logsumexp(l)                          (Alg. 1)
  grads by reverse mode through the energy and both encoders; one Adam step (A-15).
Under data parallelism (north_star) the oracle runs on the GLOBAL batch (rank-ordered
concatenation of the local batches, A-21), i.e. the gradient of the global mean loss.

Actor (Eq. 3, §5.1 P:313 "tuneable entropy coefficient", App. C alpha = 0):
  [mu, log_sigma] = pi_enc([s || g]),  log_sigma clipped to [-5, 2]  (paper silent; A-27)
  u = mu + sigma * eps,  a' = tanh(u)
  log pi = sum_k (-eps_k^2/2 - log sigma_k - log(2 pi)/2) - sum_k log(1 - a'_k^2 + 1e-6)
  L_actor = (1/N) sum_i (alpha_ent log pi_i - f(phi([s_i || a'_i]), psi(g_i)))
  differentiated w.r.t. the actor parameters only (critic frozen).

Entropy coefficient ("a tuneable entropy coefficient"; the paper gives no rule,
reading A-32 takes SAC's automatic tuning):
  L_alpha = alpha (-mean_i log pi_i - H_target),  alpha = exp(log_alpha),
  one Adam step (oracle/adam.py, no weight decay) on log_alpha with gradient L_alpha.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from . import adam, energy, losses, mlp


def split_critic_params(flat, obs_dim, act_dim, goal_dim, depth, width, repr_dim, layernorm=False):
    flat = np.asarray(flat, np.float64)
    up = mlp.unpack_ln if layernorm else mlp.unpack
    phi_layers, n_phi = up(flat, obs_dim + act_dim, depth, width, repr_dim)
    psi_layers, n_psi = up(flat[n_phi:], goal_dim, depth, width, repr_dim)
    assert n_phi + n_psi == flat.size, (n_phi, n_psi, flat.size)
    return phi_layers, psi_layers


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as fp64 (diagnostic emulate_bf16 only)."""
    x32 = np.asarray(x, np.float32)
    b = x32.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def critic_forward_backward(params, s, a, g, *, obs_dim, act_dim, goal_dim, depth, width,
                            repr_dim, energy_kind="l2", loss_kind="sym", beta=0.1,
                            activation="silu", layernorm=False):
    """Everything up to (not including) the optimiser.  Returns a dict.  layernorm: the F2
    encoders (LayerNorm before every hidden activation, oracle/mlp.py)."""
    phi_layers, psi_layers = split_critic_params(params, obs_dim, act_dim, goal_dim, depth,
                                                 width, repr_dim, layernorm)
    fwd, bwd, pk = (mlp.forward_ln, mlp.backward_ln, mlp.pack_ln) if layernorm else \
        (mlp.forward, mlp.backward, mlp.pack)
    x_phi = np.concatenate([np.asarray(s, np.float64), np.asarray(a, np.float64)], axis=1)
    x_psi = np.asarray(g, np.float64)
    Phi, cache_phi = fwd(phi_layers, x_phi, activation)
    Psi, cache_psi = fwd(psi_layers, x_psi, activation)
    l = energy.logits(energy_kind, Phi, Psi)
    comps, G = losses.loss_and_grad(l, loss_kind, beta)
    dPhi, dPsi = energy.vjp(energy_kind, Phi, Psi, G)
    g_phi, _ = bwd(phi_layers, cache_phi, dPhi, activation)
    g_psi, _ = bwd(psi_layers, cache_psi, dPsi, activation)
    grads = np.concatenate([pk(g_phi), pk(g_psi)])
    return dict(comps, phi=Phi, psi=Psi, logits=l, dlogits=G, dphi=dPhi, dpsi=dPsi, grads=grads)


def critic_step(params, m, v, t, s, a, g, *, lr=3e-4, b1=0.9, b2=0.999, eps=1e-8, wd=0.0,
                **kw):
    """C7: forward + loss + backward + Adam.  Returns the dict of critic_forward_backward
    plus params_new, m_new, v_new, t_new."""
    out = critic_forward_backward(params, s, a, g, **kw)
    p2, m2, v2, t2 = adam.adam_step(params, out["grads"], m, v, t, lr, b1, b2, eps, wd)
    out.update(params_new=p2, m_new=m2, v_new=v2, t_new=t2)
    return out


# ----------------------------------------------------------------------------------------
# Actor loss (C8)
# ----------------------------------------------------------------------------------------

LOG_SIG_MIN, LOG_SIG_MAX = -5.0, 2.0


def _energy_diag_grad_phi(kind, phi, psi):
    """d f(phi_i, psi_i) / d phi_i, row by row."""
    if kind == "dot":
        return psi.copy()
    if kind == "l2":
        r = np.sqrt(((phi - psi) ** 2).sum(1) + energy.EPS_L2)
        return -(phi - psi) / r[:, None]
    if kind == "cos":
        npsi = np.maximum(np.linalg.norm(psi, axis=1), energy.EPS_COS)
        v = psi / npsi[:, None]
        return energy._cos_back(phi, v)
    if kind == "l2sq":
        return -2.0 * (phi - psi)
    if kind == "l1":
        return -np.sign(phi - psi)
    raise ValueError(kind)


def tanh_gaussian_sample_log_prob(mu, log_sig, eps_noise):
    """The policy of Eq. 3 as a tanh-squashed diagonal Gaussian (reading A-27 for
    the clip, done by the caller): u = mu + sigma eps, a' = tanh(u) and, by the change of
    variables a' = tanh(u) (du/da' = 1 / (1 - tanh(u)^2)),
        log pi(a') = sum_k [log N(u_k; mu_k, sigma_k^2)] - sum_k log(1 - a'_k^2 + 1e-6)
                   = sum_k (-eps_k^2/2 - log sigma_k - log(2 pi)/2) - sum_k log(1 - a'_k^2 + 1e-6)
    (log N(u; mu, sigma^2) = -(u - mu)^2 / (2 sigma^2) - log sigma - log(2 pi)/2 with
    (u - mu) / sigma = eps; the 1e-6 keeps the log finite as |a'| -> 1).
    Returns (a' [N][act], log pi [N])."""
    mu = np.asarray(mu, np.float64); log_sig = np.asarray(log_sig, np.float64)
    eps_noise = np.asarray(eps_noise, np.float64)
    sig = np.exp(log_sig)
    u = mu + sig * eps_noise
    a_new = np.tanh(u)
    log_pi = (-0.5 * eps_noise ** 2 - log_sig - 0.5 * np.log(2 * np.pi)).sum(1) \
        - np.log(1.0 - a_new ** 2 + 1e-6).sum(1)
    return a_new, log_pi


def actor_loss(actor_params, critic_params, s, g, eps_noise, *, alpha_ent, obs_dim, act_dim,
               goal_dim, depth, width, repr_dim, actor_depth=2, actor_width=256,
               energy_kind="l2", activation="silu"):
    """Returns dict(loss, grads (actor, flat), a_new, log_pi, f_diag)."""
    s = np.asarray(s, np.float64); g = np.asarray(g, np.float64)
    eps_noise = np.asarray(eps_noise, np.float64)
    N = s.shape[0]
    pi_layers, n_pi = mlp.unpack(actor_params, obs_dim + goal_dim, actor_depth, actor_width,
                                 2 * act_dim)
    assert n_pi == np.asarray(actor_params).size
    phi_layers, psi_layers = split_critic_params(critic_params, obs_dim, act_dim, goal_dim,
                                                 depth, width, repr_dim)
    out, cache_pi = mlp.forward(pi_layers, np.concatenate([s, g], axis=1), activation)
    mu, log_sig_raw = out[:, :act_dim], out[:, act_dim:]
    log_sig = np.clip(log_sig_raw, LOG_SIG_MIN, LOG_SIG_MAX)
    sig = np.exp(log_sig)
    a_new, log_pi = tanh_gaussian_sample_log_prob(mu, log_sig, eps_noise)
    Phi, cache_phi = mlp.forward(phi_layers, np.concatenate([s, a_new], axis=1), activation)
    Psi, _ = mlp.forward(psi_layers, g, activation)
    f = energy.diag_logits(energy_kind, Phi, Psi)
    loss = np.mean(alpha_ent * log_pi - f)
    # reverse mode
    dPhi = -(1.0 / N) * _energy_diag_grad_phi(energy_kind, Phi, Psi)
    _, dX = mlp.backward(phi_layers, cache_phi, dPhi, activation)
    da = dX[:, obs_dim:]
    one_m = 1.0 - a_new ** 2
    du = da * one_m + (alpha_ent / N) * 2.0 * a_new * one_m / (one_m + 1e-6)
    dmu = du
    dlog_sig = du * sig * eps_noise - alpha_ent / N
    inside = (log_sig_raw >= LOG_SIG_MIN) & (log_sig_raw <= LOG_SIG_MAX)
    dlog_sig_raw = np.where(inside, dlog_sig, 0.0)
    g_pi, _ = mlp.backward(pi_layers, cache_pi, np.concatenate([dmu, dlog_sig_raw], axis=1),
                           activation)
    return dict(loss=loss, grads=mlp.pack(g_pi), a_new=a_new, log_pi=log_pi, f_diag=f)


def entropy_update(log_pi, log_alpha, m, v, t, *, target_entropy, lr, b1=0.9, b2=0.999, eps=1e-8):
    """One step of the entropy-coefficient tuning (reading A-32).  log_pi: the GLOBAL batch's
    log pi (mean taken here).  Returns dict(log_alpha, alpha, loss, m, v, t)."""
    alpha = np.exp(np.float64(log_alpha))
    loss = alpha * (-np.mean(np.asarray(log_pi, np.float64)) - target_entropy)
    # d/dlog_alpha [exp(log_alpha) c] = exp(log_alpha) c = loss
    p, m, v, t = adam.adam_step(np.array([log_alpha], np.float64), np.array([loss]), np.array([m]),
                                np.array([v]), t, lr=lr, b1=b1, b2=b2, eps=eps, wd=0.0)
    return dict(log_alpha=float(p[0]), alpha=float(np.exp(p[0])), loss=float(loss), m=float(m[0]),
                v=float(v[0]), t=t)
