"""Trajectory replay buffer and hindsight relabeling — oracle (contract C1 in DESIGN.md).

Paper passages followed:
  * Alg. 1 P:1030-1038 — per-env trajectories of (s, a, s'); on a terminal s' the env
    resets and a new trajectory starts;
  * Table 2 P:918-919 + P:928-929 — max_replay_size is *per environment* (capacity T);
  * P:165-169 (§3) — goals are "the state T steps in the future for T ~ Geom(1-gamma)";
  * P:190-191, P:219 (§3.1, §3.2) — (s, a) sampled uniformly, g from the states that
    occur *after* s in the same trajectory;
  * Alg. 1 P:1045-1046 — "randomly sample (with discount) a batch".
Readings: A-07 offset k >= 1; A-08 truncated + renormalised geometric
over the L in-episode successors present; A-09 goal = goal-slice of the state stored at
tau+k; A-10 starts with no successor rejected deterministically (attempt counter in the
Philox counter, cap 64); A-11 uniform = multiply-shift of a 32-bit word; A-12 goal slice
obs[goal_offset : goal_offset+goal_dim]; A-18 Philox4x32-10.

This oracle keeps the FULL history per env with absolute step indices and finds the
episode end by a linear scan of the done flags.  It knows nothing about rings or
per-slot metadata (the GPU path's data structures).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from .philox import philox4x32_10

MAX_ATTEMPTS = 64
TWO64 = 1 << 64


class SamplerError(RuntimeError):
    """All 64 attempts drew a start with no in-episode successor (A-10)."""


class OracleBuffer:
    """Per-env history of (obs, act, done) indexed by absolute step; capacity T per env."""

    def __init__(self, n_envs, obs_dim, act_dim, capacity):
        self.E, self.obs_dim, self.act_dim, self.T = n_envs, obs_dim, act_dim, capacity
        self.obs = [[] for _ in range(n_envs)]
        self.act = [[] for _ in range(n_envs)]
        self.done = [[] for _ in range(n_envs)]
        self.n_ins = 0

    def insert(self, obs, act, done):
        """obs[U][E][obs_dim], act[U][E][act_dim], done[U][E] (time-major, Alg. 1 loop order)."""
        U = obs.shape[0]
        for u in range(U):
            for e in range(self.E):
                self.obs[e].append(np.asarray(obs[u, e], np.float32).copy())
                self.act[e].append(np.asarray(act[u, e], np.float32).copy())
                self.done[e].append(int(done[u, e]))
        self.n_ins += U

    def window(self):
        """(tau_old, tau_new, n): the absolute indices still stored (last T inserted)."""
        tau_new = self.n_ins - 1
        tau_old = max(0, self.n_ins - self.T)
        return tau_old, tau_new, tau_new - tau_old + 1

    def successors_in_episode(self, e, tau):
        """L = min(tau*, tau_new) - tau with tau* the first tau' >= tau whose done flag is 1.

        Linear scan of the done flags (the plain definition)."""
        _, tau_new, _ = self.window()
        d = self.done[e]
        t = tau
        while t <= tau_new:
            if d[t] == 1:
                return t - tau
            t += 1
        return tau_new - tau


def geometric_tables(gamma, T):
    """G[k] = gamma^k by repeated fp64 multiplication, k = 0..T; Q[k] = floor((1-G[k]) 2^64)
    (saturated at 2^64-1).  Q[k]/2^64 is the CDF of Geom(1-gamma) on {1..k}:
    P(K <= k) = 1 - gamma^k."""
    G = [1.0]
    for _ in range(T):
        G.append(G[-1] * gamma)
    Q = []
    for g in G:
        x = 1.0 - g
        Q.append(TWO64 - 1 if x >= 1.0 else int(x * 18446744073709551616.0))
    return G, Q


def offset_from_uniform(R, L, Q):
    """k = min{k in [1, L] : Q[k] > t}, t = floor(R * Q[L] / 2^64): inverse-CDF sampling of the
    geometric law truncated to [1, L] and renormalised (A-08).  R is a uniform 64-bit word."""
    t = (R * Q[L]) >> 64
    for k in range(1, L + 1):
        if Q[k] > t:
            return k
    raise AssertionError("unreachable: t < Q[L]")


def exact_offset_pmf(L, Q):
    """The exact law the integer procedure realises: P(k) = (Q[k] - Q[k-1]) / Q[L]."""
    return np.array([(Q[k] - Q[k - 1]) / Q[L] for k in range(1, L + 1)], dtype=np.float64)


def relabel_sample(buf: OracleBuffer, seed, step, batch_local, rank=0, world=1, gamma=0.99,
                   goal_offset=0, goal_dim=2, Q=None, rows=None):
    """Hindsight relabel sample of ``batch_local`` rows for rank ``rank`` (C1).

    Returns s[B_l][obs], a[B_l][act], g[B_l][goal] (fp32 copies) and idx[B_l][3] int64 =
    (global env, tau, tau+k) with absolute step indices.  ``rows`` (optional) restricts the
    computation to those local rows (others stay zero) — every row is independent.

    These are the critic's goals (always hindsight goals); the random-goal mixture of App. C
    applies to the actor's goals only: see ``random_goal_mix``.
    """
    tau_old, tau_new, n = buf.window()
    if n < 2:
        raise SamplerError("buffer holds fewer than 2 slots per env")
    if Q is None:
        _, Q = geometric_tables(gamma, buf.T)
    E_l = buf.E
    s = np.zeros((batch_local, buf.obs_dim), np.float32)
    a = np.zeros((batch_local, buf.act_dim), np.float32)
    g = np.zeros((batch_local, goal_dim), np.float32)
    idx = np.zeros((batch_local, 3), np.int64)
    seed_lo, seed_hi = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    step_lo, step_hi = step & 0xFFFFFFFF, (step >> 32) & 0xFFFFFFFF
    for r in (range(batch_local) if rows is None else rows):
        rho = rank * batch_local + r                       # global row id
        for att in range(MAX_ATTEMPTS):
            x0, x1, x2, x3 = (int(v) for v in philox4x32_10(rho, att, step_lo, step_hi, seed_lo, seed_hi))
            e = (x0 * E_l) >> 32                            # uniform env (A-11)
            j = (x1 * n) >> 32                              # uniform slot among the n stored
            tau = tau_old + j
            L = buf.successors_in_episode(e, tau)
            if L >= 1:
                break
        else:
            raise SamplerError(f"row {rho}: {MAX_ATTEMPTS} attempts without a valid start")
        R = (x2 << 32) | x3
        k = offset_from_uniform(R, L, Q)
        s[r] = buf.obs[e][tau]
        a[r] = buf.act[e][tau]
        g[r] = buf.obs[e][tau + k][goal_offset:goal_offset + goal_dim]
        idx[r] = (rank * E_l + e, tau, tau + k)
    return s, a, g, idx


def random_goal_mix(buf: OracleBuffer, seed, step, batch_local, g, alpha, rank=0, goal_offset=0,
                    goal_dim=2, rows=None):
    """The actor's goals under random-goal mixing (F4; App. C P:951-964 mixes random goals into
    the POLICY objective only, reading A-36).  Starting from the hindsight goals ``g`` of the
    same (seed, step) sample: with the draw (y0..y3) = Philox(rho, 64, step) (attempt counter
    64, past the 0..63 start attempts of ``relabel_sample``), a row whose
    y0 < floor(alpha 2^32) takes the goal slice of a uniformly random stored state: env
    (y1 E_l) >> 32, slot tau_old + ((y2 n) >> 32).  alpha is taken at fp32 precision (the ABI
    field).  Returns (g_actor fp32 [B_l][goal_dim], flagged bool [B_l])."""
    tau_old, tau_new, n = buf.window()
    E_l = buf.E
    g_actor = np.array(g, np.float32, copy=True)
    flagged = np.zeros(batch_local, bool)
    seed_lo, seed_hi = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    step_lo, step_hi = step & 0xFFFFFFFF, (step >> 32) & 0xFFFFFFFF
    thr = int(float(np.float32(alpha)) * 4294967296.0)
    if thr == 0:
        return g_actor, flagged
    for r in (range(batch_local) if rows is None else rows):
        rho = rank * batch_local + r
        y0, y1, y2, _ = (int(v) for v in philox4x32_10(rho, MAX_ATTEMPTS, step_lo, step_hi, seed_lo, seed_hi))
        if y0 < thr:
            e2 = (y1 * E_l) >> 32
            t2 = tau_old + ((y2 * n) >> 32)
            g_actor[r] = buf.obs[e2][t2][goal_offset:goal_offset + goal_dim]
            flagged[r] = True
    return g_actor, flagged


def relabel_sample_sharded(bufs, seed, step, batch_local, **kw):
    """W-shard semantics (C1): rank r samples from its own buffer (global envs
    [r E_l, (r+1) E_l)); the global batch is the rank-ordered concatenation."""
    outs = [relabel_sample(b, seed, step, batch_local, rank=r, world=len(bufs), **kw)
            for r, b in enumerate(bufs)]
    return tuple(np.concatenate([o[i] for o in outs]) for i in range(4))
