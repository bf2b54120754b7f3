"""World size 2 on real GPUs (north_star's data-parallel critic step): two ranks,
one GPU each, NCCL over NVLink through the library's own communicator, global negatives
(every rank's phi_i against all of psi).  The concatenation of the ranks'
local batches is the global batch the fp64 oracle sees; the all-reduced loss and gradient
and the post-Adam parameters are compared with it, and must be identical across ranks.

Skipped when fewer than two GPUs are visible (the round-end GPU tier has one), so the first
multi-GPU run checks correctness before it is timed."""
import multiprocessing as mp

import numpy as np
import pytest

import crl_synth
from _crl_testlib import make_ctx, oracle_kw, rel, relmax

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _two_gpus():
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.device_count() >= 2
    except Exception:
        return False


def _rank_main(rank, world, cfg, nccl_id, q):
    try:
        import torch
        torch.cuda.set_device(rank)
        ctx, params = make_ctx(cfg, world=world, rank=rank, nccl_id=nccl_id)
        Bl = cfg["batch"] // world
        s, a, g = crl_synth.random_batch(cfg, cfg["batch"], seed=11)
        sl = slice(rank * Bl, (rank + 1) * Bl)
        loss = torch.zeros(4, device="cuda")
        grads = torch.zeros(ctx.n_params, device="cuda")
        ctx.critic_step(torch.from_numpy(s[sl]).cuda(), torch.from_numpy(a[sl]).cuda(),
                        torch.from_numpy(g[sl]).cuda(), loss, grads)
        torch.cuda.synchronize()
        q.put((rank, ctx.status(), loss.cpu().numpy(), grads.cpu().numpy(), ctx.params.cpu().numpy(),
               ctx.debug_tensor("lse_row").cpu().numpy(), None))
    except Exception as e:                      # report, do not hang the parent
        q.put((rank, -1, None, None, None, None, repr(e)))


@pytest.mark.skipif(not _two_gpus(), reason="needs 2 GPUs")
@pytest.mark.parametrize("preset,prec,batch,extra", [
    ("ant", "fp32", 512, {}),
    ("ant", "bf16", 2200, {}),
    ("ant", "bf16", 1200, {"width": 256, "repr_dim": 256}),
])
def test_critic_step_world2(preset, prec, batch, extra):
    from oracle import critic as ocritic
    from paper_2408_11052_b200 import nccl_unique_id
    cfg = crl_synth.preset(preset, precision=prec, batch=batch, **extra)
    nid = nccl_unique_id()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_rank_main, args=(r, 2, cfg, nid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert res[r][6] is None, res[r][6]
        assert res[r][1] == 0, f"rank {r} status {res[r][1]}"
    params = crl_synth.init_critic_params(cfg, 42).astype(np.float64)
    s, a, g = crl_synth.random_batch(cfg, batch, seed=11)
    z = np.zeros_like(params)
    ref = ocritic.critic_step(params, z, z, 0, s, a, g, lr=cfg["lr"], **oracle_kw(cfg))
    tol = BF16_TOL if prec == "bf16" else 1e-4
    Bl = batch // 2
    for r in range(2):
        L = res[r][2]
        for i, k in enumerate(["L_fwd", "L_bwd", "penalty", "total"]):
            assert abs(L[i] - ref[k]) <= tol * max(abs(ref[k]), 1e-3), (r, k, L[i], ref[k])
        assert rel(res[r][3], ref["grads"]) < tol, r
        assert relmax(res[r][3], ref["grads"]) < 5 * tol, r
        assert rel(res[r][5], ref["lse_row"][r * Bl:(r + 1) * Bl]) < tol, r
    # data parallelism keeps the replicas in lock step: same all-reduced gradient, same update
    assert np.array_equal(res[0][3], res[1][3])
    assert np.array_equal(res[0][4], res[1][4])
