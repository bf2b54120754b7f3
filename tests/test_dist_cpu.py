"""Multi-rank (world size 2, gloo, CPU) tests of the data-parallel decomposition the CUDA path
uses, checked against the single-process oracle on the global batch.

Per rank r (rows [r B_l, (r+1) B_l), envs [r E_l, (r+1) E_l)):
  sample its rows from its own buffer shard -> local Phi_l, Psi_l -> all-gather Phi, Psi
  LSE_l = row LSE of (Phi_l vs Psi_g), LSE'_l = row LSE of (Psi_l vs Phi_g)  (two-call design);
  or (one-pass, L2 / cos) column sums of e^l over the local rows, all-reduced, log   (C2)
  all-gather LSE, LSE'; all-reduce the 3 loss partial sums
  dPhi_l from rows of dL/dl (needs LSE'_g), dPsi_l from the transposed problem (needs LSE_g)
  local encoder backward -> all-reduce (sum) of the gradients
The result must equal the oracle critic step on the concatenated global batch (A-21, A-23).
Also: the NCCL unique-id bootstrap broadcast and the per-rank workspace sizing of the ABI.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import crl_synth

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_rows(x):
    parts = [torch.zeros_like(torch.from_numpy(x)) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(x)))
    return torch.cat(parts).numpy()


def _worker(rank, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import critic, energy, losses, mlp, replay

        chunks = crl_synth.fast_chunks(cfg, 3, U=40)
        loc = crl_synth.rank_chunks(chunks, rank, WORLD)
        buf = replay.OracleBuffer(cfg["n_envs"] // WORLD, cfg["obs_dim"], cfg["act_dim"], cfg["capacity"])
        for c in loc:
            buf.insert(*c)
        Bl = cfg["batch"] // WORLD
        N = cfg["batch"]
        s, a, g, idx = replay.relabel_sample(buf, 77, 3, Bl, rank=rank, world=WORLD, gamma=cfg["gamma"],
                                             goal_dim=cfg["goal_dim"])
        kw = dict(obs_dim=cfg["obs_dim"], act_dim=cfg["act_dim"], goal_dim=cfg["goal_dim"],
                  depth=cfg["depth"], width=cfg["width"], repr_dim=cfg["repr_dim"])
        params = crl_synth.init_critic_params(cfg, 5).astype(np.float64)
        phi_l, psi_l = critic.split_critic_params(params, **kw)
        Phi_l, cphi = mlp.forward(phi_l, np.concatenate([s, a], 1).astype(np.float64))
        Psi_l, cpsi = mlp.forward(psi_l, g.astype(np.float64))
        Phi_g, Psi_g = _gather_rows(Phi_l), _gather_rows(Psi_l)
        E, beta = cfg["energy"], cfg["beta_lse"]
        # pass 1: the two row-owner LSE calls
        l_rows = energy.logits(E, Phi_l, Psi_g)                 # [B_l][N]
        l_cols_T = energy.logits(E, Psi_l, Phi_g)               # [B_l][N] = columns of l, transposed
        lse_l = losses.lse_rows(l_rows)
        lsec_l = losses.lse_rows(l_cols_T)
        lse_g, lsec_g = _gather_rows(lse_l), _gather_rows(lsec_l)
        # one-pass statistics at W > 1 (the bounded energies): this rank's
        # column sums of e^l over its rows for ALL N columns, all-reduced, then log
        colsum = torch.from_numpy(np.exp(l_rows).sum(0))
        dist.all_reduce(colsum)
        lsec_onepass = np.log(colsum.numpy())
        diag = energy.diag_logits(E, Phi_l, Psi_l)
        acc = torch.tensor([np.sum(lse_l - diag), np.sum(lsec_l - diag), np.sum(lse_l ** 2)])
        dist.all_reduce(acc)
        L_fwd, L_bwd, P = acc[0].item() / N, acc[1].item() / N, beta * acc[2].item() / N
        # pass 2: rows of dL/dl for this rank's phi rows, and for its psi rows (transposed)
        rows = rank * Bl + np.arange(Bl)
        I_rows = (rows[:, None] == np.arange(N)[None, :]).astype(np.float64)
        p = np.exp(l_rows - lse_l[:, None])
        q = np.exp(l_rows - lsec_g[None, :])
        G_rows = (p - I_rows + q - I_rows) / N + (2 * beta / N) * lse_l[:, None] * p
        pT = np.exp(l_cols_T - lse_g[None, :])                 # p_ji seen from psi row j
        qT = np.exp(l_cols_T - lsec_l[:, None])
        GT_rows = (pT - I_rows + qT - I_rows) / N + (2 * beta / N) * lse_g[None, :] * pT
        dPhi_l, _ = energy.vjp(E, Phi_l, Psi_g, G_rows)
        dPsi_l, _ = energy.vjp(E, Psi_l, Phi_g, GT_rows)        # f is symmetric in its arguments
        g_phi, _ = mlp.backward(phi_l, cphi, dPhi_l)
        g_psi, _ = mlp.backward(psi_l, cpsi, dPsi_l)
        grads = torch.from_numpy(np.concatenate([mlp.pack(g_phi), mlp.pack(g_psi)]))
        dist.all_reduce(grads)
        # NCCL unique-id bootstrap through torch.distributed (host logic of bootstrap_nccl_id)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        out_q.put((rank, dict(L_fwd=L_fwd, L_bwd=L_bwd, P=P, grads=grads.numpy(), idx=idx, s=s, a=a, g=g,
                              id_ok=obj[0] == bytes(range(128)), lsec_onepass=lsec_onepass,
                              lsec_local=lsec_l)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("energy_kind", ["l2", "dot", "cos", "l1", "l2sq"])
def test_dp_decomposition_matches_global_oracle(energy_kind):
    cfg = crl_synth.preset("reacher", batch=24, width=16, depth=2, repr_dim=16, n_envs=4, capacity=80,
                           energy=energy_kind, beta_lse=0.1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, cfg, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import critic, replay
    chunks = crl_synth.fast_chunks(cfg, 3, U=40)
    bufs = []
    for r in range(WORLD):
        b = replay.OracleBuffer(cfg["n_envs"] // WORLD, cfg["obs_dim"], cfg["act_dim"], cfg["capacity"])
        for c in crl_synth.rank_chunks(chunks, r, WORLD):
            b.insert(*c)
        bufs.append(b)
    s, a, g, idx = replay.relabel_sample_sharded(bufs, 77, 3, cfg["batch"] // WORLD, gamma=cfg["gamma"],
                                                 goal_dim=cfg["goal_dim"])
    assert np.array_equal(np.concatenate([res[0]["idx"], res[1]["idx"]]), idx)
    params = crl_synth.init_critic_params(cfg, 5).astype(np.float64)
    ref = critic.critic_forward_backward(params, s, a, g, obs_dim=cfg["obs_dim"], act_dim=cfg["act_dim"],
                                         goal_dim=cfg["goal_dim"], depth=cfg["depth"], width=cfg["width"],
                                         repr_dim=cfg["repr_dim"], energy_kind=energy_kind, loss_kind="sym",
                                         beta=0.1)
    for r in range(WORLD):
        assert abs(res[r]["L_fwd"] - ref["L_fwd"]) < 1e-12
        assert abs(res[r]["L_bwd"] - ref["L_bwd"]) < 1e-12
        assert abs(res[r]["P"] - ref["penalty"]) < 1e-12
        assert np.allclose(res[r]["grads"], ref["grads"], rtol=1e-9, atol=1e-12)
        assert res[r]["id_ok"]
        # C2: the all-reduced one-pass column statistics equal the two-call column LSEs of this
        # rank's columns and, for every column, the global oracle's (no running max needed for
        # L2 / cos: e^l <= e)
        if energy_kind in ("l2", "cos"):
            Bl = cfg["batch"] // WORLD
            assert np.allclose(res[r]["lsec_onepass"][r * Bl:(r + 1) * Bl], res[r]["lsec_local"], rtol=1e-12, atol=1e-12)
            assert np.allclose(res[r]["lsec_onepass"], ref["lse_col"], rtol=1e-12, atol=1e-12)


def test_abi_per_rank_workspace_and_validation():
    from paper_2408_11052_b200 import CrlConfig, CrlError, workspace_size
    cfg = crl_synth.preset("ant")
    sizes = [workspace_size(CrlConfig.from_preset(cfg, world_size=4, rank=r)) for r in range(4)]
    assert all(s == sizes[0] for s in sizes)             # ranks are symmetric
    one = workspace_size(CrlConfig.from_preset(cfg))
    # rings shard by env; each rank keeps its own offset table (T+1 u64) and alignment slack
    assert sizes[0]["buffer_bytes"] * 4 <= one["buffer_bytes"] + 4 * (8 * 1001 + 5 * 256)
    bad = CrlConfig.from_preset(cfg, world_size=2, rank=2)
    with pytest.raises(CrlError):
        workspace_size(bad)
