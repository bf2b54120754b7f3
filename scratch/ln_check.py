# Development check (not a test): per-tensor gradient errors of bf16 critic steps vs the oracle
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import crl_synth
from oracle import critic as ocritic
from test_gpu_parity import make_ctx, oracle_kw, param_tensors
from _crl_testlib import rel

def run(**kw):
    cfg = crl_synth.preset(kw.pop("preset"), **kw)
    ctx, params = make_ctx(cfg)
    B = cfg["batch"]
    s, a, g = crl_synth.random_batch(cfg, B, seed=11)
    loss = torch.zeros(4, device="cuda"); grads = torch.zeros(ctx.n_params, device="cuda")
    ctx.critic_step(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(), torch.from_numpy(g).cuda(), loss, grads)
    torch.cuda.synchronize()
    z = np.zeros_like(params, dtype=np.float64)
    ref = ocritic.critic_step(params.astype(np.float64), z, z, 0, s, a, g, lr=cfg["lr"], **oracle_kw(cfg))
    gr = grads.cpu().numpy(); off = 0; out = []
    for name, n in param_tensors(cfg):
        out.append(f"{name}:{rel(gr[off:off+n], ref['grads'][off:off+n]):.3g}"); off += n
    print(kw, "dphi", f"{rel(ctx.debug_tensor('dphi').cpu().numpy(), ref['dphi']):.3g}", " ".join(out))

for c in [dict(preset="ant", precision="bf16", batch=512, width=512, activation="relu", layernorm=1),
          dict(preset="ant", precision="bf16", batch=512, width=512, activation="silu", layernorm=1),
          dict(preset="ant", precision="bf16", batch=512, width=512, activation="relu", layernorm=0),
          dict(preset="ant", precision="bf16", batch=640, width=256, activation="silu", layernorm=1),
          dict(preset="ant", precision="bf16", batch=640, width=256, activation="relu", layernorm=1)]:
    run(**c)
