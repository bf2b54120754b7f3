"""Shared helpers for the GPU parity tests: build a context from a preset, fill its buffer
with synthetic trajectories (crl_synth), and run the oracle on the same inputs."""
import numpy as np

import crl_synth


def oracle_kw(cfg):
    return dict(obs_dim=cfg["obs_dim"], act_dim=cfg["act_dim"], goal_dim=cfg["goal_dim"],
                depth=cfg["depth"], width=cfg["width"], repr_dim=cfg["repr_dim"],
                energy_kind=cfg["energy"], loss_kind=cfg["loss"], beta=cfg["beta_lse"],
                activation=cfg["activation"], layernorm=bool(cfg.get("layernorm", 0)))


def rel(a, b):
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def relmax(a, b):
    """Element-wise companion of rel(): max_k |a_k - b_k| / max_k |b_k| (SURVEY 8(c) parity
    metric: a wrong ragged block or a single bad element cannot hide under a norm)."""
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def param_tensors(cfg):
    """(name, size) of every parameter tensor in the flat critic layout (include/crl.h): per
    encoder (phi, then psi) and layer W[in][out], b[out] and, on LayerNorm hidden layers (F2),
    gamma[out], beta[out]."""
    ln = bool(cfg.get("layernorm", 0))
    out = []
    for enc, enc_in in (("phi", cfg["obs_dim"] + cfg["act_dim"]), ("psi", cfg["goal_dim"])):
        for li, (fi, fo) in enumerate(crl_synth.param_shapes(enc_in, cfg["depth"], cfg["width"], cfg["repr_dim"])):
            out += [(f"{enc}.W{li}", fi * fo), (f"{enc}.b{li}", fo)]
            if ln and li < cfg["depth"]:
                out += [(f"{enc}.ln_gamma{li}", fo), (f"{enc}.ln_beta{li}", fo)]
    return out


def make_ctx(cfg, world=1, rank=0, nccl_id=None, seed=42, **over):
    import torch
    from paper_2408_11052_b200 import CrlConfig, CrlContext
    c = CrlConfig.from_preset(cfg, world_size=world, rank=rank, **over)
    params = crl_synth.init_critic_params(cfg, seed)
    ctx = CrlContext(c, params=torch.from_numpy(params), nccl_id=nccl_id)
    return ctx, params


def fill_buffer(ctx, cfg, n_chunks=3, U=None, world=1, rank=0, seed=1234):
    """Insert synthetic chunks into the GPU buffer; returns the (global) host chunks."""
    import torch
    chunks = crl_synth.fast_chunks(cfg, n_chunks, U=U, seed=seed)
    local = crl_synth.rank_chunks(chunks, rank, world)
    for obs, act, done in local:
        ctx.buffer_insert(torch.from_numpy(obs).cuda(), torch.from_numpy(act).cuda(),
                          torch.from_numpy(done).cuda())
    return chunks


def oracle_buffers(cfg, chunks, world=1):
    from oracle import replay
    bufs = []
    for r in range(world):
        loc = crl_synth.rank_chunks(chunks, r, world)
        b = replay.OracleBuffer(cfg["n_envs"] // world, cfg["obs_dim"], cfg["act_dim"], cfg["capacity"])
        for obs, act, done in loc:
            b.insert(obs, act, done)
        bufs.append(b)
    return bufs
