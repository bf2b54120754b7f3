"""CPU checks of the C ABI boundary: libcrl.so loads, exports every symbol include/crl.h
declares, and its host-only logic (workspace sizing, argument validation) behaves.  No
compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

import crl_synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2408_11052_b200 import load_library
    return load_library()


def declared_symbols():
    with open(os.path.join(ROOT, "include", "crl.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"CRL_API\s+[\w\s\*]+?\b(crl_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["crl_buffer_insert", "crl_relabel_sample", "crl_critic_step", "crl_actor_loss"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = _lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    from paper_2408_11052_b200 import EXPORTED
    assert sorted(EXPORTED) == declared_symbols()
    assert lib.crl_abi_version() == 3


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {os.path.join(ROOT, 'paper_2408_11052_b200', 'libcrl.so')}").read()
    assert "sm_100a" in out, out[:500]


@pytest.mark.parametrize("name", ["reacher", "ant", "humanoid", "sweep4096"])
def test_workspace_size_param_count(name):
    from paper_2408_11052_b200 import CrlConfig, workspace_size
    cfg = crl_synth.preset(name, precision="fp32")
    ws = workspace_size(CrlConfig.from_preset(cfg))
    assert ws["n_params"] == crl_synth.critic_param_count(cfg)
    assert ws["buffer_bytes"] >= cfg["n_envs"] * cfg["capacity"] * 4 * (cfg["obs_dim"] + cfg["act_dim"])
    assert ws["scratch_bytes"] % 256 == 0


def test_paper_param_counts():
    # 168,576 / 438,144 / 501,888 / 6,864,384 params
    assert crl_synth.critic_param_count(crl_synth.preset("reacher")) == 168576
    assert crl_synth.critic_param_count(crl_synth.preset("ant")) == 438144
    assert crl_synth.critic_param_count(crl_synth.preset("humanoid")) == 501888
    assert crl_synth.critic_param_count(crl_synth.preset("netscale")) == 6864384


@pytest.mark.parametrize("over,code", [
    (dict(batch_local=1), 1),                 # N < 2: no negatives
    (dict(gamma=1.0), 1),                     # gamma must be < 1
    (dict(repr_dim=48), 7),                   # unsupported D
    (dict(goal_offset=28), 1),                # goal slice out of range
    (dict(rank=1), 1),                        # rank >= world
])
def test_workspace_size_validation(over, code):
    from paper_2408_11052_b200 import CrlConfig, CrlError, workspace_size
    cfg = CrlConfig.from_preset(crl_synth.preset("ant"))
    for k, v in over.items():
        setattr(cfg, k, v)
    with pytest.raises(CrlError) as ei:
        workspace_size(cfg)
    assert ei.value.code == code


def test_sharded_workspace_is_smaller_per_rank():
    from paper_2408_11052_b200 import CrlConfig, workspace_size
    cfg = crl_synth.preset("ant")
    one = workspace_size(CrlConfig.from_preset(cfg))
    two = workspace_size(CrlConfig.from_preset(cfg, world_size=2, rank=1))
    assert two["buffer_bytes"] < one["buffer_bytes"]
    assert two["n_params"] == one["n_params"]


def test_layernorm_param_count_matches_library():
    """F2: the library's n_params for LayerNorm encoders equals the documented layout (W, b,
    gamma, beta per hidden layer)."""
    from paper_2408_11052_b200 import CrlConfig, workspace_size
    cfg = crl_synth.preset("netscale", precision="fp32", batch=256, layernorm=1)
    ws = workspace_size(CrlConfig.from_preset(cfg))
    assert ws["n_params"] == crl_synth.critic_param_count(cfg)
    assert ws["n_params"] == crl_synth.critic_param_count(dict(cfg, layernorm=0)) + 2 * 2 * 4 * 1024
