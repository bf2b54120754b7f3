"""Pins for oracle/philox.py and oracle/replay.py (contract C1), CPU only.

Pins: Random123 KAT vectors; the integer offset law vs the closed-form truncated geometric
PMF (A-08); chi-square of sampled offsets and of (env, slot) uniformity;
exhaustive boundary audit (A-09); special cases gamma = 0 and L = 1; ring window
after wrap-around; W-shard semantics (A-21)."""
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle.philox import philox4x32_10
from oracle import replay
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_philox_known_answer_vectors():
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        vals = [int(x, 16) for x in r]
        out = philox4x32_10(*vals[:6])
        assert [int(x) for x in out] == vals[6:]


def test_philox_vectorised_matches_scalar():
    c = np.arange(100, dtype=np.uint64)
    vec = philox4x32_10(c, c * 3, 7, 9, 0xDEADBEEF, 0x12345678)
    for i in (0, 17, 99):
        sc = philox4x32_10(int(c[i]), int(c[i]) * 3, 7, 9, 0xDEADBEEF, 0x12345678)
        assert [int(v[i]) for v in vec] == [int(x) for x in sc]


@pytest.mark.parametrize("gamma", [0.0, 0.5, 0.9, 0.99])
@pytest.mark.parametrize("L", [1, 2, 7, 100, 1000])
def test_offset_pmf_matches_truncated_geometric(gamma, L):
    _, Q = replay.geometric_tables(gamma, 1000)
    pmf = replay.exact_offset_pmf(L, Q)
    k = np.arange(1, L + 1)
    if gamma == 0.0:
        ref = (k == 1).astype(float)
    else:
        ref = gamma ** (k - 1) * (1 - gamma) / (1 - gamma ** L)
    assert np.max(np.abs(pmf - ref)) <= 1e-12
    assert abs(pmf.sum() - 1.0) <= 1e-12


def test_offset_pmf_paper_value(closed_forms):
    _, Q = replay.geometric_tables(0.99, 1000)
    pmf = replay.exact_offset_pmf(1000, Q)
    assert abs(pmf[0] - closed_forms["offset_p1_g099_L1000"]) < 1e-12


def test_offset_special_cases():
    _, Q0 = replay.geometric_tables(0.0, 50)
    rng = np.random.default_rng(0)
    for R in [0, (1 << 64) - 1] + [int(x) for x in rng.integers(0, 2**63, 50)]:
        assert replay.offset_from_uniform(R, 37, Q0) == 1        # gamma = 0 => k = 1
    _, Q = replay.geometric_tables(0.99, 50)
    for R in [0, (1 << 64) - 1, 12345]:
        assert replay.offset_from_uniform(R, 1, Q) == 1          # L = 1 => k = 1
    assert replay.offset_from_uniform(0, 40, Q) == 1              # smallest word -> k = 1
    assert replay.offset_from_uniform((1 << 64) - 1, 40, Q) == 40  # largest word -> k = L


@pytest.mark.parametrize("gamma,L", [(0.9, 30), (0.99, 1000), (0.5, 7)])
def test_offset_histogram_chi_square(gamma, L):
    _, Q = replay.geometric_tables(gamma, 1000)
    rng = np.random.default_rng(123)
    n = 100_000
    words = rng.integers(0, 2**63, n, dtype=np.uint64).astype(object) * 2 + rng.integers(0, 2, n).astype(object)
    ks = np.array([replay.offset_from_uniform(int(R), L, Q) for R in words])
    pmf = replay.exact_offset_pmf(L, Q)
    counts = np.bincount(ks, minlength=L + 1)[1:]
    exp = pmf * n
    # merge the tail into bins with expected count >= 5
    obs_b, exp_b, acc_o, acc_e = [], [], 0, 0.0
    for o, e in zip(counts, exp):
        acc_o += o; acc_e += e
        if acc_e >= 5:
            obs_b.append(acc_o); exp_b.append(acc_e); acc_o, acc_e = 0, 0.0
    if acc_e > 0:
        obs_b[-1] += acc_o; exp_b[-1] += acc_e
    p = stats.chisquare(obs_b, exp_b).pvalue
    assert p > 0.01, p


def _buffer_from_done(done_2d, obs_dim=3, act_dim=2, T=None, seed=0):
    """done_2d[E][steps] -> OracleBuffer with obs[e][t] = (e, t, noise...)."""
    E, S = done_2d.shape
    rng = np.random.default_rng(seed)
    buf = replay.OracleBuffer(E, obs_dim, act_dim, T or S)
    obs = np.zeros((S, E, obs_dim), np.float32)
    obs[:, :, 0] = np.arange(E)[None, :]
    obs[:, :, 1] = np.arange(S)[:, None]
    obs[:, :, 2:] = rng.standard_normal((S, E, obs_dim - 2))
    act = rng.uniform(-1, 1, (S, E, act_dim)).astype(np.float32)
    buf.insert(obs, act, done_2d.T.copy())
    return buf


def test_relabel_gamma0_goal_is_next_state():
    done = np.zeros((2, 12), np.uint8); done[0, 4] = 1; done[1, 7] = 1
    buf = _buffer_from_done(done)
    s, a, g, idx = replay.relabel_sample(buf, seed=5, step=3, batch_local=200, gamma=0.0,
                                         goal_dim=2)
    assert np.all(idx[:, 2] == idx[:, 1] + 1)
    assert np.all(g[:, 1] == idx[:, 2])          # obs[...,1] stores the absolute step
    assert np.all(g[:, 0] == idx[:, 0])          # same env


def test_relabel_boundary_audit_and_uniform_starts():
    rng = np.random.default_rng(1)
    E, S, T = 4, 90, 60                          # wraps: only the last 60 steps are stored
    done = (rng.random((E, S)) < 0.08).astype(np.uint8)
    buf = _buffer_from_done(done, T=T)
    tau_old, tau_new, n = buf.window()
    assert (tau_old, tau_new, n) == (30, 89, 60)
    B = 4000
    s, a, g, idx = replay.relabel_sample(buf, seed=99, step=0, batch_local=B, gamma=0.9)
    e, tau, tk = idx[:, 0], idx[:, 1], idx[:, 2]
    assert np.all(tau >= tau_old) and np.all(tk <= tau_new) and np.all(tk > tau)
    for r in range(B):                           # no episode end in [tau, tau+k-1]
        assert done[e[r], tau[r]:tk[r]].sum() == 0
    assert np.all(s[:, 1] == tau) and np.all(s[:, 0] == e)
    # valid starts: L >= 1; empirical frequency ~ uniform over them
    valid = [(ee, t) for ee in range(E) for t in range(tau_old, tau_new + 1)
             if buf.successors_in_episode(ee, t) >= 1]
    pos = {v: i for i, v in enumerate(valid)}
    counts = np.zeros(len(valid))
    for r in range(B):
        counts[pos[(e[r], tau[r])]] += 1
    p = stats.chisquare(counts).pvalue
    assert p > 0.001, p


def test_relabel_deterministic_and_row_independent():
    rng = np.random.default_rng(2)
    done = (rng.random((3, 40)) < 0.1).astype(np.uint8)
    buf = _buffer_from_done(done)
    full = replay.relabel_sample(buf, seed=1, step=7, batch_local=32, gamma=0.99)
    again = replay.relabel_sample(buf, seed=1, step=7, batch_local=32, gamma=0.99)
    sub = replay.relabel_sample(buf, seed=1, step=7, batch_local=32, gamma=0.99, rows=[3, 30])
    for x, y in zip(full, again):
        assert np.array_equal(x, y)
    assert np.array_equal(full[3][[3, 30]], sub[3][[3, 30]])
    other = replay.relabel_sample(buf, seed=1, step=8, batch_local=32, gamma=0.99)
    assert not np.array_equal(full[3], other[3])


def test_relabel_sharded_semantics():
    rng = np.random.default_rng(3)
    done = (rng.random((4, 50)) < 0.05).astype(np.uint8)
    b0 = _buffer_from_done(done[:2]); b1 = _buffer_from_done(done[2:])
    B_l = 16
    s, a, g, idx = replay.relabel_sample_sharded([b0, b1], seed=4, step=2, batch_local=B_l)
    r1 = replay.relabel_sample(b1, 4, 2, B_l, rank=1, world=2)
    assert np.array_equal(idx[B_l:], r1[3])
    assert np.all(idx[:B_l, 0] < 2) and np.all(idx[B_l:, 0] >= 2)   # global env ids


def test_relabel_rejects_tiny_buffer():
    done = np.zeros((2, 1), np.uint8)
    buf = _buffer_from_done(done)
    with pytest.raises(replay.SamplerError):
        replay.relabel_sample(buf, 0, 0, 4)
    done = np.ones((1, 5), np.uint8)             # every slot ends its episode: no valid start
    buf = _buffer_from_done(done)
    with pytest.raises(replay.SamplerError):
        replay.relabel_sample(buf, 0, 0, 4)


# ------------------------------------------------------------------ F4 random-goal mixing (A-36)

def test_random_goal_alpha_mixing():
    """App. C: a fraction alpha of the ACTOR's goals is the goal slice of a uniformly
    random stored state (the critic keeps the hindsight goals, reading A-36).  alpha = 0
    leaves every goal unchanged; with alpha = 0.3 the flagged fraction matches alpha
    (binomial 4-sigma band), flagged goals are stored states of the window, unflagged rows
    are the hindsight goals; alpha = 1 flags every row."""
    rng = np.random.default_rng(3)
    E, T, U = 6, 50, 70
    buf = replay.OracleBuffer(E, 4, 2, T)
    obs = rng.standard_normal((U, E, 4)).astype(np.float32)
    act = rng.standard_normal((U, E, 2)).astype(np.float32)
    done = (rng.random((U, E)) < 0.05).astype(np.uint8)
    buf.insert(obs, act, done)
    B = 2000
    base = replay.relabel_sample(buf, 77, 5, B, gamma=0.9, goal_dim=2)
    same, f0 = replay.random_goal_mix(buf, 77, 5, B, base[2], 0.0, goal_dim=2)
    assert np.array_equal(same, base[2]) and not f0.any()
    mix, flag = replay.random_goal_mix(buf, 77, 5, B, base[2], 0.3, goal_dim=2)
    assert abs(flag.mean() - 0.3) < 4 * math.sqrt(0.3 * 0.7 / B)
    assert np.array_equal(mix[~flag], base[2][~flag])
    tau_old, tau_new, _ = buf.window()
    stored = {tuple(buf.obs[e][t][:2]) for e in range(E) for t in range(tau_old, tau_new + 1)}
    assert all(tuple(gg) in stored for gg in mix[flag])
    b64 = replay.relabel_sample(buf, 77, 5, 64, gamma=0.9, goal_dim=2)
    _, fall = replay.random_goal_mix(buf, 77, 5, 64, b64[2], 1.0, goal_dim=2)
    assert fall.all()
