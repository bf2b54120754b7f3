"""F4: the collection side in the loop — env steps/s of a full CRL iteration on one GPU.

Alg. 1: collect `unroll_length` (62) steps of every env, insert them into the
replay buffer, then run gradient updates (critic + actor; Table 2).  The paper's
environments (Brax) are out of scope, so a GPU *env stand-in* produces the
transitions: a seeded random walk on the device (obs_{t+1} = obs_t + 0.1 a_t + noise, actions
N(0, 1) clipped, episodes ending with hazard 1/episode_length).  Per iteration:
  env stand-in (U x E_l steps, torch ops) -> crl_buffer_insert -> crl_relabel_sample_bulk
  (n_updates batches in one launch) -> n_updates x (crl_critic_step + crl_actor_loss with Adam)
and the line reports env steps/s (the paper's end-to-end unit) and updates/s, timed with CUDA
events on the launching stream (one JSON line, not the bench.py contract line).

    python scripts/pipeline_bench.py --workload ant --updates 16 --iters 10
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import crl_synth  # noqa: E402
from paper_2408_11052_b200 import CrlConfig, CrlContext  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="ant")
    p.add_argument("--precision", default="bf16")
    p.add_argument("--updates", type=int, default=16, help="gradient updates per collection round")
    p.add_argument("--iters", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--no-actor", action="store_true")
    args = p.parse_args()

    cfg = crl_synth.preset(args.workload, precision=args.precision)
    E, U, B = cfg["n_envs"], cfg["unroll_length"], cfg["batch"]
    O, A, G = cfg["obs_dim"], cfg["act_dim"], cfg["goal_dim"]
    actor = not args.no_actor
    over = dict(actor_depth=2, actor_width=256) if actor else {}
    ccfg = CrlConfig.from_preset(cfg, **over)
    params = crl_synth.init_critic_params(cfg, 42)
    kw = dict(actor_params=torch.from_numpy(crl_synth.init_actor_params(cfg, 43))) if actor else {}
    ctx = CrlContext(ccfg, params=torch.from_numpy(params), **kw)
    st = torch.cuda.Stream()
    gen = torch.Generator(device="cuda").manual_seed(1234)
    obs_t = torch.zeros(E, O, device="cuda")
    obs_buf = torch.empty(U, E, O, device="cuda")
    act_buf = torch.empty(U, E, A, device="cuda")
    done_buf = torch.empty(U, E, dtype=torch.uint8, device="cuda")
    nU = args.updates
    s = torch.empty(nU * B, O, device="cuda")
    a = torch.empty(nU * B, A, device="cuda")
    g = torch.empty(nU * B, G, device="cuda")
    eps = torch.empty(B, A, device="cuda")
    loss = torch.zeros(4, device="cuda")
    aloss = torch.zeros(1, device="cuda")
    hazard = 1.0 / cfg["episode_length"]
    step_ctr = [0]

    def collect():
        # the env stand-in: a device random walk in the first A coordinates, resets on done
        for u in range(U):
            act = torch.randn(E, A, device="cuda", generator=gen).clamp_(-1, 1)
            obs_buf[u] = obs_t
            act_buf[u] = act
            d = torch.rand(E, device="cuda", generator=gen) < hazard
            done_buf[u] = d.to(torch.uint8)
            nxt = obs_t.clone()
            nxt[:, :A] += 0.1 * act
            nxt += 0.01 * torch.randn(E, O, device="cuda", generator=gen)
            obs_t.copy_(torch.where(d[:, None], torch.zeros_like(nxt), nxt))

    def iteration():
        collect()
        ctx.buffer_insert(obs_buf, act_buf, done_buf, stream=st)
        ctx.relabel_sample_bulk(crl_synth.PHILOX_SEED, step_ctr[0], nU, s, a, g, stream=st)
        for k in range(nU):
            sl = slice(k * B, (k + 1) * B)
            ctx.critic_step(s[sl], a[sl], g[sl], loss, stream=st)
            if actor:
                eps.normal_(generator=gen)
                ctx.actor_loss(s[sl], g[sl], eps, 0.1, loss_out=aloss, apply_adam=True, stream=st)
        step_ctr[0] += nU

    with torch.cuda.stream(st):
        # fill the ring once (~T / U rounds) so sampling sees a full window, then warm up
        for _ in range(max(2, cfg["capacity"] // U + 1)):
            collect()
            ctx.buffer_insert(obs_buf, act_buf, done_buf, stream=st)
        for _ in range(args.warmup):
            iteration()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(args.iters):
            iteration()
        e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    env_steps = args.iters * U * E
    line = {"metric": "CRL training iteration throughput (env stand-in)", "env_steps_per_s": round(env_steps / (ms * 1e-3)),
            "updates_per_s": round(args.iters * nU / (ms * 1e-3), 1), "ms_per_iter": round(ms / args.iters, 3),
            "config": {"workload": cfg["name"], "n_envs": E, "unroll": U, "batch": B, "updates_per_round": nU,
                       "actor": actor, "precision": args.precision, "env": "GPU random-walk stand-in (torch)"},
            "status": ctx.status()}
    print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
