#!/usr/bin/env python
"""Benchmark: CRL critic update steps/s (BASELINE.json metric) on synthetic data.

A "step" is one pass of the whole hot path over one batch: crl_relabel_sample (A1) on the
HBM-resident replay buffer followed by crl_critic_step (A2-A6: encoders fwd, online-LSE
logits + loss, in-pass dlogits, encoders bwd, gradient all-reduce, fused Adam).  The buffer
is filled (A0) before the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--workload ant] [--precision fp32]
  python bench.py --impl reference ...     # the CPU oracle timed on the host cores

Default workload = BASELINE.json configs[4] at W = 1 ("netscale": Ant dims, 4x1024 encoders,
repr 256, global batch 16384, L2, symmetric InfoNCE, beta 0.1, 1024 envs x 1000, bf16): the
largest single-GPU configuration in BASELINE.json (its metric names no config) and the
strong-scaling config of the 1/2/4/8-GPU runs.  Prints ONE JSON line on rank 0.

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run (N ranks, one
per GPU, 127.0.0.1 rendezvous).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import crl_synth  # noqa: E402

METRIC = "CRL critic update steps/sec at batch B, 1/2/4/8 B200; % of HBM/tensor roofline"
UNIT = "steps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="netscale")
    p.add_argument("--precision", default="bf16")
    p.add_argument("--energy", default=None)
    p.add_argument("--loss", default=None, help="fwd / bwd / sym / flatnce_* / fb / dpo / ipo / sppo")
    p.add_argument("--layernorm", action="store_true", help="F2 LayerNorm encoders (fp32 path; bf16 at widths 256..1024)")
    p.add_argument("--profile-steps", type=int, default=20)
    p.add_argument("--sample-every", type=int, default=16,
                   help="batches sampled per crl_relabel_sample_bulk launch inside the timed steps "
                        "(Alg. 1: a collection round's updates are sampled together); 1 = one "
                        "crl_relabel_sample per step")
    p.add_argument("--bulk-updates", type=int, default=256,
                   help="A1 bulk-mode measurement: updates per crl_relabel_sample_bulk call (0: skip)")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--cpu-rows", type=int, default=1024,
                   help="cpu_baseline / reference arm: oracle sub-batch per timed step when the "
                        "workload's batch is larger (the step time is extrapolated to the full batch)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def workload_cfg(args):
    over = {}
    if args.precision:
        over["precision"] = args.precision
    if args.energy:
        over["energy"] = args.energy
    if args.loss:
        over["loss"] = args.loss
    if args.layernorm:
        over["layernorm"] = 1
    return crl_synth.preset(args.workload, **over)


def n_fill_chunks(cfg):
    # enough U=62 chunks to wrap the ring (20 chunks = 1240 steps for T=1000)
    return int(np.ceil((cfg["capacity"] * 1.24) / cfg["unroll_length"]))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def stop(self, t_lo=None, t_hi=None):
        """Samples taken in [t_lo, t_hi] (host monotonic clock around the timed region; the
        sampler runs from before the warm-up so nvidia-smi is up when timing starts).  A timed
        region shorter than one 100 ms sample period keeps the samples nearest to it."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if t_lo is not None and t_hi is not None:
            inside = [x for x in lines if t_lo <= x[0] <= t_hi + 0.1]
            if not inside and lines:                   # nearest samples around a short region
                inside = sorted(lines, key=lambda x: min(abs(x[0] - t_lo), abs(x[0] - t_hi)))[:2]
            lines = inside
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- roofline
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def stage_work(stage, cfg, N, Bl):
    """Algorithmic work of ONE launch of a stage: (amount, unit, bound)."""
    D, Wd, depth = cfg["repr_dim"], cfg["width"], cfg["depth"]
    in_phi, in_psi = cfg["obs_dim"] + cfg["act_dim"], cfg["goal_dim"]
    fp32 = cfg["precision"] == "fp32"
    dims = lambda i: [i] + [Wd] * depth + [D]
    tc_logits = (not fp32) and D in (64, 128, 256)   # csrc/ctx.h kTcLogitsMinN
    if stage in ("lse_fused", "grad_fused"):
        # one-pass statistics (tc_stats.cu) / one-pass gradient (tc_gradf.cu): every logit once,
        # MUFU ops per logit = 2 for L2 (rsqrt + exp2), 1 for dot / cos (exp2) -- the
        # algorithmic count of SURVEY §8(d) D3 (4 resp. 2 per step over the two passes)
        return Bl * N * (2.0 if cfg["energy"] == "l2" else 1.0), "op", "xu"
    if stage == "grad_pair":
        # D = 256 gradient pass (tc_grad2p.cu, both sides in one launch): the algorithmic work is
        # the two contractions dPhi = W Psi, dPsi = W^T Phi (2 x 2 N_l N D flops) -- the S
        # recompute the kernel also does is NOT counted -- and 2 MUFU ops per logit (L2); at
        # D = 256 the tensor term binds
        return 4.0 * Bl * N * D, "flop", "tensor"
    if stage in ("dw_db_grouped", "dw_db_pairs"):
        # every dW_l = X_l^T dZ_l of both encoders (the bias sums ride on the same tiles)
        tot = 0.0
        for ind in (in_phi, in_psi):
            d = dims(ind)
            tot += sum(2.0 * Bl * d[l] * d[l + 1] for l in range(len(d) - 1))
        return tot, "flop", "tensor"
    if stage in ("lse_row", "lse_col", "grad_phi", "grad_psi") and tc_logits:
        # bf16 path: the logits stage is bound by the MUFU/XU pipe: the
        # algorithmic transcendental count of the WHOLE stage is 4 per logit for L2 (one exp +
        # one sqrt per pass) and 2 for dot/cos; four launches share it -> 1/4 per launch.
        per = (4.0 if cfg["energy"] == "l2" else 2.0) / 4.0
        return Bl * N * per, "op", "xu"
    if stage == "lse_pair":
        # both sides' online-max statistics in one launch: half of the stage's count
        return Bl * N * (4.0 if cfg["energy"] == "l2" else 2.0) / 2.0, "op", "xu"
    if stage in ("lse_row", "lse_col"):
        # fp32 path: the logits GEMM (2 N^2 D, counted once for both orientations) -> N_l N D
        return Bl * N * D * 1.0, "flop", "alu"
    if stage in ("grad_phi", "grad_psi"):
        # the two backward contractions (W Psi and W^T Phi): 2 N^2 D each, one per launch
        return 2.0 * Bl * N * D, "flop", "alu"
    if stage in ("mlp_fwd_chain", "mlp_bwd_chain", "mlp_fwd_cchain", "mlp_bwd_cchain"):
        # fused chains (per-row-block or cluster-split): every layer of both encoders
        # (forward), every dX step (backward)
        tot = 0.0
        for ind in (in_phi, in_psi):
            d = dims(ind)
            rng = range(len(d) - 1) if stage.startswith("mlp_fwd") else range(1, len(d) - 1)
            tot += sum(2.0 * Bl * d[l] * d[l + 1] for l in rng)
        return tot, "flop", "tensor"
    if stage == "rowstat":
        return float(2 * Bl * D * 2), "byte", "hbm"
    if stage == "prep_inputs":
        return float(Bl * (in_phi + in_psi) * 6), "byte", "hbm"
    if "_bwd_db_" in stage:
        out = D if stage.endswith(f"_l{depth}") else Wd
        return float(Bl * out * 2), "byte", "hbm"
    if stage == "adam":
        return 28.0 * crl_synth.critic_param_count(cfg), "byte", "hbm"
    if stage == "relabel":
        row = 4 * (2 * (cfg["obs_dim"] + cfg["act_dim"] + cfg["goal_dim"])) + 4
        return float(row * Bl), "byte", "hbm"
    if stage == "loss":
        return float(Bl * D * 4 * 2), "byte", "hbm"
    if stage.startswith("enc_fwd_l") or stage.startswith("enc_bwd_dx_l"):
        # one CTA-pair launch for layer l of BOTH encoders (tc_pgemm2)
        l = int(stage.rsplit("_l", 1)[1])
        return sum(2.0 * Bl * dims(ind)[l] * dims(ind)[l + 1] for ind in (in_phi, in_psi)), "flop", "tensor"
    for tag, ind in (("phi", in_phi), ("psi", in_psi)):
        if stage.startswith(tag + "_"):
            l = int(stage.rsplit("_l", 1)[1])
            d = dims(ind)
            return 2.0 * Bl * d[l] * d[l + 1], "flop", "alu" if fp32 else "tensor"
    return None, None, None


def roofline(stages, cfg, N, Bl, peaks, peak_kind, clocks, traffic_db, step_ms=0.0):
    known = {k: v for k, v in stages.items() if stage_work(k, cfg, N, Bl)[0] is not None}
    if "lse_fused" in stages:
        # lse_pair (lse_row / lse_col) is then the exact fallback, gated off by a device flag (early exit)
        known.pop("lse_row", None)
        known.pop("lse_col", None)
        known.pop("lse_pair", None)
    if not known:
        return None                      # --profile-steps 0: no per-stage measurement
    name, (ms, cnt) = max(known.items(), key=lambda kv: kv[1][0])
    per_launch_ms = ms / cnt
    work, unit, bound = stage_work(name, cfg, N, Bl)
    if bound == "hbm":
        achieved = work / (per_launch_ms * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        u = "GB/s"
        note = f"HBM copy bandwidth ({peak_kind} MEASURED_PEAKS.json hbm_gbs)"
    elif bound == "tensor":
        achieved = work / (per_launch_ms * 1e-3) / 1e12
        # a kernel timed inside a long step (>= 1 ms of back-to-back tensor work: the clocks sit
        # at the power cap) is held to the sustained peak, a short one to the burst peak
        sustained = step_ms >= 1.0 and "bf16_tflops_sustained" in peaks
        peak = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
        u = "TFLOP/s"
        note = (f"dense bf16 ({peak_kind} MEASURED_PEAKS.json "
                f"{'bf16_tflops_sustained: timed inside a >= 1 ms step' if sustained else 'bf16_tflops, burst'})")
    elif bound == "xu":
        # MUFU/XU transcendental pipe: 148 SMs x 16 ops/clk x clock
        mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        achieved = work / (per_launch_ms * 1e-3) / 1e9
        peak = 148 * 16 * mhz * 1e6 / 1e9
        u = "Gop/s"
        bound = "alu"
        note = f"MUFU/XU pipe: 148 SM x 16 op/clk x {mhz:.0f} MHz (median SM clock under load)"
    else:
        # fp32 SIMT: 148 SMs x 128 FP32 lanes x 2 flop/FMA x clock
        mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        achieved = work / (per_launch_ms * 1e-3) / 1e12
        peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
        u = "TFLOP/s"
        note = f"FP32 FMA pipe: 148 SM x 128 lanes x 2 x {mhz:.0f} MHz (median SM clock under load)"
    return {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": u,
            "frac": round(achieved / peak, 4), "traffic": traffic_db.get(name),
            "kernel": name, "launch_us": round(per_launch_ms * 1e3, 3),
            "share_of_step": round(ms / max(1e-9, sum(v[0] for v in stages.values())), 4),
            "peak_source": note,
            "stages_us": {k: round(v[0] / v[1] * 1e3, 2) for k, v in stages.items()}}


# ----------------------------------------------------------------------------- CPU oracle
def host_info():
    """CPU model and NumPy's BLAS vendor (BASELINE.md §4 asks for both next to the cores)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        b = [x for x in threadpool_info() if x.get("user_api") == "blas"]
        if b:
            blas = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('num_threads')} threads)"
    except Exception:
        pass
    return model, blas


def oracle_steps(cfg, chunks, seconds, max_steps, seed_step0=0, warm=1, rows=1024):
    """Time the oracle critic step (relabel + fwd + loss + bwd + Adam) on the host cores.

    At batch N <= rows every timed step is one whole oracle step.  Above it (the net-scale and
    large sweep configs: the fp64 oracle's N x N logits would take minutes per step) each timed
    step runs the oracle's stages on an n = rows sub-batch drawn from the same workload, and
    the full-batch step time is extrapolated from the stages' measured times with their exact
    scaling in N:  t(N) = (t_relabel + t_encoders)(N/n) + t_logits (N/n)^2 + t_adam
    (relabel and both encoders are per-row; energies, loss and VJP are N x N; Adam is per
    parameter).  Returns (steps/s at N, threads, timed steps, description)."""
    from threadpoolctl import threadpool_info

    from oracle import adam as oadam
    from oracle import critic as ocritic
    from oracle import energy as oenergy
    from oracle import losses as olosses
    from oracle import mlp as omlp
    from oracle import replay as oreplay
    buf = oreplay.OracleBuffer(cfg["n_envs"], cfg["obs_dim"], cfg["act_dim"], cfg["capacity"])
    for obs, act, done in chunks:
        buf.insert(obs, act, done)
    _, Q = oreplay.geometric_tables(cfg["gamma"], cfg["capacity"])
    params = crl_synth.init_critic_params(cfg, 42).astype(np.float64)
    m = np.zeros_like(params); v = np.zeros_like(params); t = 0
    ln = bool(cfg.get("layernorm", 0))
    kw = dict(obs_dim=cfg["obs_dim"], act_dim=cfg["act_dim"], goal_dim=cfg["goal_dim"],
              depth=cfg["depth"], width=cfg["width"], repr_dim=cfg["repr_dim"],
              energy_kind=cfg["energy"], loss_kind=cfg["loss"], beta=cfg["beta_lse"],
              activation=cfg["activation"], layernorm=ln)
    B = cfg["batch"]
    n = min(B, rows)
    scale = B / n
    times = []
    step = seed_step0
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        s, a, g, _ = oreplay.relabel_sample(buf, crl_synth.PHILOX_SEED, step, n, gamma=cfg["gamma"],
                                            goal_dim=cfg["goal_dim"], Q=Q)
        t1 = time.perf_counter()
        if n == B:
            out = ocritic.critic_step(params, m, v, t, s, a, g, lr=cfg["lr"], **kw)
            params, m, v, t = out["params_new"], out["m_new"], out["v_new"], out["t_new"]
            times.append(time.perf_counter() - t0)
        else:
            # the same stages as oracle/critic.py critic_forward_backward + critic_step, timed apart
            phi_l, psi_l = ocritic.split_critic_params(params, cfg["obs_dim"], cfg["act_dim"], cfg["goal_dim"],
                                                       cfg["depth"], cfg["width"], cfg["repr_dim"], ln)
            fwd, bwd, pk = (omlp.forward_ln, omlp.backward_ln, omlp.pack_ln) if ln else \
                (omlp.forward, omlp.backward, omlp.pack)
            Phi, c_phi = fwd(phi_l, np.concatenate([s, a], axis=1).astype(np.float64), cfg["activation"])
            Psi, c_psi = fwd(psi_l, np.asarray(g, np.float64), cfg["activation"])
            t2 = time.perf_counter()
            lg = oenergy.logits(cfg["energy"], Phi, Psi)
            _, G = olosses.loss_and_grad(lg, cfg["loss"], cfg["beta_lse"])
            dPhi, dPsi = oenergy.vjp(cfg["energy"], Phi, Psi, G)
            t3 = time.perf_counter()
            g_phi, _ = bwd(phi_l, c_phi, dPhi, cfg["activation"])
            g_psi, _ = bwd(psi_l, c_psi, dPsi, cfg["activation"])
            grads = np.concatenate([pk(g_phi), pk(g_psi)])
            t4 = time.perf_counter()
            params, m, v, t = oadam.adam_step(params, grads, m, v, t, cfg["lr"], 0.9, 0.999, 1e-8, 0.0)
            t5 = time.perf_counter()
            times.append((t1 - t0 + t2 - t1 + t4 - t3) * scale + (t3 - t2) * scale * scale + (t5 - t4))
        step += 1
        n_timed = len(times) - warm
        if n_timed >= max_steps or (n_timed >= 1 and time.perf_counter() - t_start > seconds):
            break
    timed = times[warm:] if len(times) > warm else times
    blas = [x for x in threadpool_info() if x.get("user_api") == "blas"]
    cores = blas[0]["num_threads"] if blas else 1
    if n == B:
        desc = f"{len(timed)} full oracle critic steps (relabel+fwd+loss+bwd+Adam, fp64 NumPy) at batch {B}"
    else:
        desc = (f"{len(timed)} oracle critic steps (relabel+fwd+loss+bwd+Adam, fp64 NumPy) on {n}-row "
                f"sub-batches of the {cfg['name']} workload, each extrapolated to batch {B} from its "
                f"stage times: (relabel + encoders) x {scale:g} + (energies + loss + VJP) x {scale * scale:g} + Adam")
    return len(timed) / sum(timed), cores, len(timed), desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workload_cfg(args)
    chunks = crl_synth.fast_chunks(cfg, n_fill_chunks(cfg))
    # each step is one oracle critic step (sub-batched + extrapolated above --cpu-rows); the
    # whole run is bounded by --cpu-seconds (at least one timed step after the warm-up)
    steps = max(1, args.steps)
    budget = max(args.cpu_seconds, 1.0)
    val, cores, n, desc = oracle_steps(cfg, chunks, budget, steps, warm=args.warmup, rows=args.cpu_rows)
    model, blas = host_info()
    line = {"metric": METRIC, "value": round(val, 6), "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": n, "warmup": args.warmup,
            "ms_per_step": round(1e3 / val, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "global_batch": cfg["batch"],
                       "energy": cfg["energy"], "loss": cfg["loss"]},
            "cpu_baseline": {"value": round(val, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "cpu_model": model, "blas": blas, "sample": desc},
            "e2e": {"value": round(val, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def step_bound_us(cfg, N, Bl, peaks):
    """SURVEY §8(d) D3 algorithmic-work bound of one step on one GPU (µs), with this box's
    MEASURED_PEAKS: encoders 2 (2 fwd + dX) MACs per row on the sustained bf16 peak (FP32 SIMT
    for fp32), logits max(6 B_l N D flops on the tensor pipe, 4 (L2) / 2 MUFU ops per logit on
    148 x 16 op/clk at the max SM clock), sampler and Adam bytes on HBM."""
    D, Wd, depth = cfg["repr_dim"], cfg["width"], cfg["depth"]
    fp32 = cfg["precision"] == "fp32"
    fwd = dx = 0
    for ind in (cfg["obs_dim"] + cfg["act_dim"], cfg["goal_dim"]):
        d = [ind] + [Wd] * depth + [D]
        fwd += sum(d[l] * d[l + 1] for l in range(len(d) - 1))
        dx += sum(d[l] * d[l + 1] for l in range(1, len(d) - 1))
    mhz = peaks.get("sm_max_mhz", 1965.0)
    tc = (148 * 128 * 2 * mhz * 1e6) if fp32 else peaks["bf16_tflops_sustained"] * 1e12
    t_enc = 2.0 * (2 * fwd + dx) * Bl / tc
    t_ltc = 6.0 * Bl * N * D / tc
    t_mufu = Bl * N * (4.0 if cfg["energy"] == "l2" else 2.0) / (148 * 16 * mhz * 1e6)
    row = 2 * 4 * (cfg["obs_dim"] + cfg["act_dim"] + cfg["goal_dim"]) + 4
    t_samp = row * Bl / (peaks["hbm_gbs"] * 1e9)
    t_adam = (28.0 if fp32 else 30.0) * crl_synth.critic_param_count(cfg) / (peaks["hbm_gbs"] * 1e9)
    return {"bound_us": round(1e6 * (t_enc + max(t_ltc, t_mufu) + t_samp + t_adam), 2),
            "encoders_us": round(1e6 * t_enc, 2), "logits_tensor_us": round(1e6 * t_ltc, 2),
            "logits_mufu_us": round(1e6 * t_mufu, 2), "sampler_us": round(1e6 * t_samp, 3),
            "adam_us": round(1e6 * t_adam, 2)}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2408_11052_b200 import CrlConfig, CrlContext, bootstrap_nccl_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's communicator-init lines (ranks, nRanks, NVLS / channels) on stderr, so a run's
        # log shows every rank joined; stdout stays the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload_cfg(args)
    N = cfg["batch"]
    if N % world:
        raise SystemExit(f"global batch {N} not divisible by {world}")
    Bl = N // world
    ccfg = CrlConfig.from_preset(cfg, world_size=world, rank=rank)
    nccl_id = bootstrap_nccl_id() if world > 1 else None
    params = crl_synth.init_critic_params(cfg, 42)
    ctx = CrlContext(ccfg, params=torch.from_numpy(params), nccl_id=nccl_id)
    stream = torch.cuda.Stream()
    chunks = crl_synth.fast_chunks(cfg, n_fill_chunks(cfg))
    with torch.cuda.stream(stream):
        for obs, act, done in crl_synth.rank_chunks(chunks, rank, world):
            ctx.buffer_insert(torch.from_numpy(obs).cuda(), torch.from_numpy(act).cuda(),
                              torch.from_numpy(done).cuda(), stream=stream)
    nb = max(1, args.sample_every)
    s_all = torch.empty(nb * Bl, cfg["obs_dim"], device="cuda")
    a_all = torch.empty(nb * Bl, cfg["act_dim"], device="cuda")
    g_all = torch.empty(nb * Bl, cfg["goal_dim"], device="cuda")
    s, a, g = s_all[:Bl], a_all[:Bl], g_all[:Bl]
    loss = torch.zeros(4, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def step(i):
        # every step trains on its own freshly sampled batch (step counter i): with nb > 1 the
        # batches of nb consecutive steps come from one bulk launch (row u*B + r of the bulk
        # call = row r of the single call at step0 + u, bit-exact), issued at the first of them
        k = i % nb
        if nb == 1:
            ctx.relabel_sample(crl_synth.PHILOX_SEED, i, s, a, g, stream=stream)
        elif k == 0:
            ctx.relabel_sample_bulk(crl_synth.PHILOX_SEED, i, nb, s_all, a_all, g_all, stream=stream)
        sl = slice(k * Bl, (k + 1) * Bl)
        ctx.critic_step(s_all[sl], a_all[sl], g_all[sl], loss, stream=stream)

    clk = ClockSampler(local)                      # nvidia-smi up before the timed region
    clk.start()
    for i in range(max(args.warmup, nb)):          # every slice's graph captured before timing
        step(i)
    launches_per_step = 1.0 / nb + ctx.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_lo = time.monotonic()
    t0 = -(-max(args.warmup, nb) // nb) * nb       # timed steps start on a bulk boundary
    n_bulk = sum(1 for i in range(args.steps) if nb > 1 and (t0 + i) % nb == 0)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()                         # L2 flush between timed iterations
            ev0[i].record(stream)
            step(t0 + i)
            ev1[i].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop(t_lo, time.monotonic())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per = [e0.elapsed_time(e1) for e0, e1 in zip(ev0, ev1)]
    total_ms = sum(per)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t)
    status = ctx.status()
    value = args.steps / (total_ms * 1e-3)

    # ---- end to end: host (pinned) batch in, host loss out, through crl_critic_step, timed by
    # the host wall clock over K back-to-back calls (the call a user makes: each one copies its
    # step's s, a, g from page-locked host memory and writes the loss into page-locked host
    # memory; the clock stops after the device has finished the last step)
    e2e = None
    if not args.no_e2e:
        K = max(3, min(args.steps, 200))
        hb = []
        for i in range(K):
            ctx.relabel_sample(crl_synth.PHILOX_SEED, 10_000_000 + i, s, a, g, stream=stream)
            torch.cuda.synchronize()
            hb.append(tuple(x.cpu().pin_memory() for x in (s, a, g)))
        hloss = torch.zeros(4).pin_memory()
        for i in range(3):
            ctx.critic_step(*hb[i % K], hloss, stream=stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for i in range(K):
            ctx.critic_step(*hb[i], hloss, stream=stream)
        stream.synchronize()
        e_ms = (time.perf_counter() - w0) * 1e3
        if world > 1:
            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t)
        e2e = {"value": round(K / (e_ms * 1e-3), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(sum(x.numel() * 4 for x in hb[0])),
               "d2h_bytes_per_step": 16, "steps": K,
               "note": "host wall clock over K back-to-back crl_critic_step calls with page-locked host "
                       "s/a/g (H2D inside each call: one DMA copy on the copy engine into the staging "
                       "set the previous call does not read, so it overlaps that call's kernels) and "
                       "a page-locked host loss written every step; no L2 flush between calls; "
                       "max over ranks"}

    # ---- per-stage profile (eager, event-bracketed) for the roofline
    ctx.profile_enable(True)
    with torch.cuda.stream(stream):
        for i in range(args.profile_steps):
            flush.zero_()
            step(20_000_000 + i)
    torch.cuda.synchronize()
    stages = ctx.profile_read()
    ctx.profile_enable(False)

    # ---- A1 in bulk mode (F4): many updates' rows in one launch, HBM fraction of the gather
    bulk = None
    if rank == 0 and args.bulk_updates > 0:
        nbu = args.bulk_updates
        bs = torch.empty(nbu * Bl, cfg["obs_dim"], device="cuda")
        ba = torch.empty(nbu * Bl, cfg["act_dim"], device="cuda")
        bg = torch.empty(nbu * Bl, cfg["goal_dim"], device="cuda")
        bi = torch.empty(nbu * Bl, 3, dtype=torch.int64, device="cuda")
        with torch.cuda.stream(stream):
            for i in range(3):
                ctx.relabel_sample_bulk(crl_synth.PHILOX_SEED, 40_000_000 + i * nbu, nbu, bs, ba, bg, bi, stream=stream)
            b0 = [torch.cuda.Event(enable_timing=True) for _ in range(10)]
            b1 = [torch.cuda.Event(enable_timing=True) for _ in range(10)]
            for i in range(10):
                flush.zero_()
                b0[i].record(stream)
                ctx.relabel_sample_bulk(crl_synth.PHILOX_SEED, 41_000_000 + i * nbu, nbu, bs, ba, bg, bi, stream=stream)
                b1[i].record(stream)
        torch.cuda.synchronize()
        us = sum(x.elapsed_time(y) for x, y in zip(b0, b1)) / 10 * 1e3
        # algorithmic bytes per row: read s, a, g + the ep_end word, write s, a, g
        # and the three int64 indices
        row_bytes = 2 * 4 * (cfg["obs_dim"] + cfg["act_dim"] + cfg["goal_dim"]) + 4 + 24
        gbs = nbu * Bl * row_bytes / (us * 1e-6) / 1e9
        peaks_b, _ = load_peaks()
        hbm = peaks_b.get("hbm_gbs") if isinstance(peaks_b, dict) else None
        bulk = {"rows": nbu * Bl, "n_updates": nbu, "us": round(us, 2), "bytes_per_row": row_bytes,
                "achieved_GBs": round(gbs, 1), "hbm_peak_GBs": hbm,
                "frac": round(gbs / hbm, 4) if hbm else None,
                "note": "crl_relabel_sample_bulk: one launch for n_updates batches (L2 flushed before each)"}

    if rank == 0:
        peaks, kind = load_peaks()
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic_db = json.load(f).get(f"{cfg['name']}/{cfg['precision']}", {})
        except Exception:
            traffic_db = {}
        rl = roofline(stages, cfg, N, Bl, peaks, kind, clocks, traffic_db, step_ms=total_ms / args.steps)
        if rl is not None:
            # the small-batch regime is bound by the chain of dependent launches, not by a unit:
            # the measured graph floor (scratch/graph_floor.cu: ~1.1 us per dependent PDL kernel
            # on B200) times this step's launches, against the measured step time
            floor = 1.1 * launches_per_step
            rl["latency"] = {"launches_per_step": launches_per_step, "graph_floor_us_per_launch": 1.1,
                             "floor_us": round(floor, 2),
                             "frac": round(floor / (total_ms / args.steps * 1e3), 4),
                             "source": "scratch/graph_floor.cu (dependent tiny kernels, CUDA graph + PDL)"}
        if rl is not None:
            # the whole step against the SURVEY §8(d) D3 bound (the north_star's roofline target)
            sb = step_bound_us(cfg, N, Bl, peaks)
            step_us = total_ms / args.steps * 1e3
            rl["step"] = dict(sb, measured_us=round(step_us, 2), frac=round(sb["bound_us"] / step_us, 4),
                              note="bound = encoders + max(logits tensor, logits MUFU) + sampler + Adam "
                                   "(SURVEY 8(d) D3, MEASURED_PEAKS sustained bf16 / HBM, MUFU at sm_max_mhz); "
                                   "frac = bound / measured step")
        cpu = None
        if not args.no_cpu_baseline:
            val, cores, n, desc = oracle_steps(cfg, chunks, args.cpu_seconds, 10_000, rows=args.cpu_rows)
            model, blas = host_info()
            cpu = {"value": round(val, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                   "cpu_model": model, "blas": blas,
                   "sample": f"{desc}; ~{args.cpu_seconds:.0f} s budget"}
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(total_ms / args.steps, 5), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32" if cfg["precision"] == "fp32" else "bf16", "data": "synthetic",
                "config": {"workload": cfg["name"], "global_batch": N, "batch_local": Bl,
                           "obs_dim": cfg["obs_dim"], "act_dim": cfg["act_dim"],
                           "goal_dim": cfg["goal_dim"], "encoders": f"{cfg['depth']}x{cfg['width']}",
                           "repr_dim": cfg["repr_dim"], "energy": cfg["energy"], "loss": cfg["loss"],
                           "beta_lse": cfg["beta_lse"], "layernorm": int(cfg.get("layernorm", 0)),
                           "buffer": f"{cfg['n_envs']}x{cfg['capacity']}",
                           "parallelism": f"dp{world}", "l2_flush": "256 MiB memset between timed steps",
                           "sampling": ("one crl_relabel_sample per step" if nb == 1 else
                                        f"crl_relabel_sample_bulk: {nb} steps' batches per launch, inside the timed steps")},
                "clocks": clocks, "e2e": e2e,
                "gpu_launches": int(round((launches_per_step - 1.0 / nb) * args.steps)) + (n_bulk if nb > 1 else args.steps),
                "gpu_launches_per_step": launches_per_step, "roofline": rl, "relabel_bulk": bulk,
                "cpu_baseline": cpu,
                "device_status": status}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) started without torchrun: become N ranks (one per GPU) via
    torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
