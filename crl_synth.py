"""Seeded synthetic inputs shared by the oracle-side tests, the GPU parity tests,
``bench.py`` and ``__graft_entry__.smoke()``.

This module holds NO arithmetic of the method (no sampling law, no MLP, no
energy, no loss, no optimiser).  It only produces:

* workload presets (plain dicts) restating BASELINE.json ``configs`` and
  SURVEY.md §8(d) D1;
* synthetic trajectories shaped like the paper's Reacher / Ant / Humanoid tasks
  (Table 1 P:887-906 for the termination column, Table 2 P:918-937 for
  episode_length / num_envs / unroll_length);
* seeded initial parameters (flat fp32, layout documented in include/crl.h);
* seeded random representations / batches for the logits-stage tests.

Recipe:
  obs_0 ~ N(0, I); obs_{t+1} = obs_t + 0.05 N(0, I); act ~ U(-1, 1);
  episode ends by truncation at ``episode_length`` (random per-env phase) or by
  a per-step termination hazard (Ant 1/250, Humanoid 1/100, Reacher 0);
  after a ``done`` the next observation is re-drawn from N(0, I).
"""
from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# Workload presets (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------

_BASE = dict(
    gamma=0.99,              # Table 2 "discounting" P:932
    beta_lse=0.1,            # Table 2 "logsumexp_penalty" P:942
    lr=3e-4,                 # Table 2 "critic_lr" P:939
    adam_b1=0.9, adam_b2=0.999, adam_eps=1e-8, weight_decay=0.0,
    energy="l2",             # Table 2 "energy_function L2" P:941
    loss="sym",              # Table 2 "symmetric_infonce" P:940
    activation="silu",
    goal_offset=0,
    episode_length=1000,     # Table 2
    unroll_length=62,        # Table 2
    capacity=1000,
    precision="fp32",
)

PRESETS = {
    # configs[0]: Reacher, 2x256, repr 64, batch 256, L2, sym, 8 envs x 1000
    "reacher": dict(_BASE, name="reacher", obs_dim=10, act_dim=2, goal_dim=2,
                    depth=2, width=256, repr_dim=64, batch=256, n_envs=8,
                    hazard=0.0),
    # configs[1]: Ant, 4x256, repr 64, batch 256, beta 0.1, 1024 envs x 1000
    "ant": dict(_BASE, name="ant", obs_dim=29, act_dim=8, goal_dim=2,
                depth=4, width=256, repr_dim=64, batch=256, n_envs=1024,
                hazard=1.0 / 250),
    # configs[2]: Humanoid, 4x256, batch 512, bf16 tensor-core path, 512 envs
    "humanoid": dict(_BASE, name="humanoid", obs_dim=268, act_dim=17, goal_dim=3,
                     depth=4, width=256, repr_dim=64, batch=512, n_envs=512,
                     hazard=1.0 / 100, precision="bf16"),
    # configs[4]: network scaling 4x1024, repr 256, global batch 16384
    "netscale": dict(_BASE, name="netscale", obs_dim=29, act_dim=8, goal_dim=2,
                     depth=4, width=1024, repr_dim=256, batch=16384, n_envs=1024,
                     hazard=1.0 / 250, precision="bf16"),
}


def preset(name: str, **over) -> dict:
    """Return a copy of a preset; ``sweep<N>`` gives configs[3] (Ant shapes, batch N)."""
    if name.startswith("sweep"):
        n = int(name[len("sweep"):])
        cfg = dict(PRESETS["ant"], name=name, batch=n)
    else:
        cfg = dict(PRESETS[name])
    cfg.update(over)
    return cfg


def param_shapes(in_dim: int, depth: int, width: int, out_dim: int):
    """[(fan_in, fan_out), ...] for one encoder: depth hidden layers then the output layer."""
    dims = [in_dim] + [width] * depth + [out_dim]
    return [(dims[i], dims[i + 1]) for i in range(len(dims) - 1)]


def encoder_param_count(in_dim, depth, width, out_dim, layernorm=False) -> int:
    return (sum(i * o + o for i, o in param_shapes(in_dim, depth, width, out_dim))
            + (2 * width * depth if layernorm else 0))


def critic_param_count(cfg) -> int:
    ln = bool(cfg.get("layernorm", 0))
    return (encoder_param_count(cfg["obs_dim"] + cfg["act_dim"], cfg["depth"], cfg["width"], cfg["repr_dim"], ln)
            + encoder_param_count(cfg["goal_dim"], cfg["depth"], cfg["width"], cfg["repr_dim"], ln))


# ----------------------------------------------------------------------------
# Parameters
# ----------------------------------------------------------------------------

def init_encoder(rng: np.random.Generator, in_dim, depth, width, out_dim, layernorm=False) -> np.ndarray:
    """Flat fp32: per layer W[in][out] (row-major) then b[out] (+ LayerNorm gamma[out],
    beta[out] on hidden layers when `layernorm`, F2).  W ~ U(+-1/sqrt(fan_in)),
    b ~ U(+-0.1/sqrt(fan_in)) (non-zero so bias gradients are exercised; A-14 says the
    paper is silent on initialisation); gamma ~ 1 + U(+-0.1), beta ~ U(+-0.1) (not exactly
    1 / 0, so their gradients and the gain are exercised)."""
    parts = []
    for li, (fi, fo) in enumerate(param_shapes(in_dim, depth, width, out_dim)):
        bound = 1.0 / np.sqrt(fi)
        parts.append(rng.uniform(-bound, bound, size=(fi, fo)).astype(np.float32).ravel())
        parts.append(rng.uniform(-0.1 * bound, 0.1 * bound, size=(fo,)).astype(np.float32))
        if layernorm and li < depth:
            parts.append((1.0 + rng.uniform(-0.1, 0.1, size=(fo,))).astype(np.float32))
            parts.append(rng.uniform(-0.1, 0.1, size=(fo,)).astype(np.float32))
    return np.concatenate(parts)


def init_critic_params(cfg, seed: int = 42) -> np.ndarray:
    """phi encoder params followed by psi encoder params (include/crl.h layout)."""
    rng = np.random.default_rng(seed)
    ln = bool(cfg.get("layernorm", 0))
    phi = init_encoder(rng, cfg["obs_dim"] + cfg["act_dim"], cfg["depth"], cfg["width"], cfg["repr_dim"], ln)
    psi = init_encoder(rng, cfg["goal_dim"], cfg["depth"], cfg["width"], cfg["repr_dim"], ln)
    return np.concatenate([phi, psi])


def init_actor_params(cfg, seed: int = 43, actor_width: int = 256, actor_depth: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return init_encoder(rng, cfg["obs_dim"] + cfg["goal_dim"], actor_depth, actor_width, 2 * cfg["act_dim"])


# ----------------------------------------------------------------------------
# Trajectories
# ----------------------------------------------------------------------------

def fast_chunks(cfg, n_chunks: int, U: int = None, n_envs=None, seed: int = 1234, env_offset: int = 0):
    """Vectorised variant for large E (1024 envs x 1240 steps): same recipe, one generator per
    (seed, env_offset, chunk) block.  Returns a list of (obs, act, done) chunks."""
    U = cfg["unroll_length"] if U is None else U
    E = cfg["n_envs"] if n_envs is None else n_envs
    rng0 = np.random.default_rng([seed, env_offset, 0xABCD])
    obs_cur = rng0.standard_normal((E, cfg["obs_dim"]))
    t_in_ep = rng0.integers(0, cfg["episode_length"], size=E)
    out = []
    for c in range(n_chunks):
        rng = np.random.default_rng([seed, env_offset, c])
        obs = np.empty((U, E, cfg["obs_dim"]), np.float32)
        act = rng.uniform(-1.0, 1.0, (U, E, cfg["act_dim"])).astype(np.float32)
        done = np.zeros((U, E), np.uint8)
        noise = 0.05 * rng.standard_normal((U, E, cfg["obs_dim"]))
        resets = rng.standard_normal((U, E, cfg["obs_dim"]))
        haz = rng.random((U, E)) < cfg["hazard"] if cfg["hazard"] > 0 else np.zeros((U, E), bool)
        for u in range(U):
            obs[u] = obs_cur
            t_in_ep += 1
            d = haz[u] | (t_in_ep >= cfg["episode_length"])
            done[u] = d
            t_in_ep[d] = 0
            obs_cur = np.where(d[:, None], resets[u], obs_cur + noise[u])
        out.append((obs, act, done))
    return out


def rank_chunks(chunks, rank: int, world: int):
    """Slice the env axis of global chunks for rank ``rank`` of ``world`` (envs [r E_l, (r+1) E_l))."""
    res = []
    for obs, act, done in chunks:
        E = obs.shape[1]
        El = E // world
        sl = slice(rank * El, (rank + 1) * El)
        res.append((np.ascontiguousarray(obs[:, sl]), np.ascontiguousarray(act[:, sl]),
                    np.ascontiguousarray(done[:, sl])))
    return res


# ----------------------------------------------------------------------------
# Random representations / batches for the logits-stage tests
# ----------------------------------------------------------------------------

def random_reps(N: int, D: int, seed: int = 7, scale: float = 1.0):
    rng = np.random.default_rng(seed)
    phi = (scale * rng.standard_normal((N, D))).astype(np.float32)
    psi = (scale * rng.standard_normal((N, D))).astype(np.float32)
    return phi, psi


def random_batch(cfg, N: int, seed: int = 11):
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((N, cfg["obs_dim"])).astype(np.float32)
    a = rng.uniform(-1, 1, (N, cfg["act_dim"])).astype(np.float32)
    g = rng.standard_normal((N, cfg["goal_dim"])).astype(np.float32)
    return s, a, g


PHILOX_SEED = 0x0000C0FFEE123457
