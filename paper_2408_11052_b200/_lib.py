"""Thin ctypes binding over libcrl.so (include/crl.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  PyTorch is used for device memory,
streams and the torch.distributed bootstrap of the NCCL unique id — nothing else.

There is no CPU fallback: if libcrl.so is missing or no CUDA device is present, the calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
# CRL_LIB_PATH: an alternative build of the same library (A/B measurements of compile-time
# variants, e.g. `make OUT=... BUILD=... NVFLAGS_EXTRA=-D...`); the in-tree build by default
LIB_PATH = os.environ.get("CRL_LIB_PATH") or os.path.join(_HERE, "libcrl.so")

CRL_OK, CRL_EINVAL, CRL_ESTATE, CRL_ECUDA, CRL_ENCCL, CRL_ENONFINITE, CRL_ESAMPLER, CRL_EUNSUPPORTED = range(8)
STATUS_NAMES = ["CRL_OK", "CRL_EINVAL", "CRL_ESTATE", "CRL_ECUDA", "CRL_ENCCL", "CRL_ENONFINITE",
                "CRL_ESAMPLER", "CRL_EUNSUPPORTED"]
ENERGY = {"l2": 0, "dot": 1, "cos": 2, "l1": 3, "l2sq": 4}
LOSS = {"fwd": 0, "bwd": 1, "sym": 2, "flatnce_fwd": 3, "flatnce_bwd": 4, "fb": 5, "dpo": 6, "ipo": 7,
        "sppo": 8}
ACT = {"silu": 0, "relu": 1}
PRECISION = {"fp32": 0, "bf16": 1}

EXPORTED = ["crl_abi_version", "crl_workspace_size", "crl_create", "crl_destroy",
            "crl_nccl_unique_id", "crl_buffer_insert", "crl_relabel_sample", "crl_critic_step",
            "crl_actor_loss", "crl_entropy_update", "crl_relabel_sample_bulk", "crl_relabel_sample_mixed", "crl_get_status", "crl_last_error", "crl_debug_tensor",
            "crl_last_launch_count", "crl_profile_enable", "crl_profile_read"]


class CrlError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES[code] if 0 <= code < 8 else code}: {msg}")
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [("obs_dim", ctypes.c_int), ("act_dim", ctypes.c_int), ("goal_dim", ctypes.c_int),
                ("goal_offset", ctypes.c_int), ("n_envs_local", ctypes.c_int),
                ("capacity", ctypes.c_int), ("gamma", ctypes.c_double), ("depth", ctypes.c_int),
                ("width", ctypes.c_int), ("repr_dim", ctypes.c_int), ("activation", ctypes.c_int),
                ("energy", ctypes.c_int), ("loss", ctypes.c_int), ("beta_lse", ctypes.c_float),
                ("lr", ctypes.c_float), ("adam_b1", ctypes.c_float), ("adam_b2", ctypes.c_float),
                ("adam_eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("precision", ctypes.c_int), ("batch_local", ctypes.c_int),
                ("world_size", ctypes.c_int), ("rank", ctypes.c_int),
                ("actor_depth", ctypes.c_int), ("actor_width", ctypes.c_int),
                ("lr_actor", ctypes.c_float), ("layernorm", ctypes.c_int),
                ("random_goal_alpha", ctypes.c_float)]


class _Sizes(ctypes.Structure):
    _fields_ = [("n_params", ctypes.c_size_t), ("n_actor_params", ctypes.c_size_t),
                ("buffer_bytes", ctypes.c_size_t), ("scratch_bytes", ctypes.c_size_t)]


class _Memory(ctypes.Structure):
    _fields_ = [("params", ctypes.c_void_p), ("adam_m", ctypes.c_void_p),
                ("adam_v", ctypes.c_void_p), ("actor_params", ctypes.c_void_p),
                ("actor_adam_m", ctypes.c_void_p), ("actor_adam_v", ctypes.c_void_p),
                ("buffer", ctypes.c_void_p), ("scratch", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libcrl.so once and declare the prototypes.  Raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libcrl.so not built ({path}); run __graft_entry__.build() — "
                           "there is no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, i, u64, f = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_float
    sig = {
        "crl_abi_version": (i, []),
        "crl_workspace_size": (i, [ctypes.POINTER(_Config), ctypes.POINTER(_Sizes)]),
        "crl_create": (i, [ctypes.POINTER(_Config), ctypes.POINTER(_Memory), vp, ctypes.POINTER(vp)]),
        "crl_destroy": (i, [vp]),
        "crl_nccl_unique_id": (i, [vp]),
        "crl_buffer_insert": (i, [vp, vp, vp, vp, i, vp]),
        "crl_relabel_sample": (i, [vp, u64, u64, vp, vp, vp, vp, vp]),
        "crl_relabel_sample_bulk": (i, [vp, u64, u64, i, vp, vp, vp, vp, vp]),
        "crl_relabel_sample_mixed": (i, [vp, u64, u64, i, vp, vp, vp, vp, vp, vp]),
        "crl_critic_step": (i, [vp, vp, vp, vp, vp, vp, vp]),
        "crl_actor_loss": (i, [vp, vp, vp, vp, f, vp, vp, i, vp]),
        "crl_entropy_update": (i, [vp, f, f, vp, vp, vp, vp]),
        "crl_get_status": (i, [vp, i, i]),
        "crl_last_error": (ctypes.c_char_p, [vp]),
        "crl_debug_tensor": (i, [vp, ctypes.c_char_p, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)]),
        "crl_last_launch_count": (i, [vp]),
        "crl_profile_enable": (i, [vp, i]),
        "crl_profile_read": (i, [vp, i, ctypes.c_char_p, i, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(i)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    if lib.crl_abi_version() != 3:
        raise RuntimeError("libcrl.so ABI version mismatch")
    _lib = lib
    return lib


def _check(code, ctx=None):
    if code != CRL_OK:
        lib = load_library()
        raise CrlError(code, lib.crl_last_error(ctx).decode())


@dataclass
class CrlConfig:
    """Mirror of crl_config (include/crl.h).  Names follow the paper's Table 2."""
    obs_dim: int
    act_dim: int
    goal_dim: int
    n_envs_local: int
    capacity: int = 1000
    batch_local: int = 256
    goal_offset: int = 0
    gamma: float = 0.99
    depth: int = 2
    width: int = 256
    repr_dim: int = 64
    activation: str = "silu"
    energy: str = "l2"
    loss: str = "sym"
    beta_lse: float = 0.1
    lr: float = 3e-4
    adam_b1: float = 0.9
    adam_b2: float = 0.999
    adam_eps: float = 1e-8
    weight_decay: float = 0.0
    precision: str = "fp32"
    world_size: int = 1
    rank: int = 0
    actor_depth: int = 0
    actor_width: int = 0
    lr_actor: float = 6e-4
    layernorm: int = 0
    random_goal_alpha: float = 0.0

    @classmethod
    def from_preset(cls, p: dict, **over):
        """Build from a crl_synth preset dict (global batch split over world_size)."""
        world = over.pop("world_size", 1)
        rank = over.pop("rank", 0)
        kw = dict(obs_dim=p["obs_dim"], act_dim=p["act_dim"], goal_dim=p["goal_dim"],
                  n_envs_local=p["n_envs"] // world, capacity=p["capacity"],
                  batch_local=p["batch"] // world, goal_offset=p["goal_offset"], gamma=p["gamma"],
                  depth=p["depth"], width=p["width"], repr_dim=p["repr_dim"],
                  activation=p["activation"], energy=p["energy"], loss=p["loss"],
                  beta_lse=p["beta_lse"], lr=p["lr"], adam_b1=p["adam_b1"], adam_b2=p["adam_b2"],
                  adam_eps=p["adam_eps"], weight_decay=p["weight_decay"],
                  precision=p["precision"], world_size=world, rank=rank,
                  layernorm=int(p.get("layernorm", 0)))
        kw.update(over)
        return cls(**kw)

    def _c(self) -> _Config:
        c = _Config()
        for name, _ in _Config._fields_:
            v = getattr(self, name)
            if name == "activation": v = ACT[v]
            elif name == "energy": v = ENERGY[v]
            elif name == "loss": v = LOSS[v]
            elif name == "precision": v = PRECISION[v]
            setattr(c, name, v)
        return c


def workspace_size(cfg: CrlConfig) -> dict:
    lib = load_library()
    s = _Sizes()
    _check(lib.crl_workspace_size(ctypes.byref(cfg._c()), ctypes.byref(s)))
    return dict(n_params=s.n_params, n_actor_params=s.n_actor_params,
                buffer_bytes=s.buffer_bytes, scratch_bytes=s.scratch_bytes)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class CrlContext:
    """Owns the device memory (torch tensors) of one crl_ctx and exposes the four hot-path
    calls under their C names."""

    def __init__(self, cfg: CrlConfig, params=None, device="cuda", nccl_id: bytes | None = None,
                 actor_params=None):
        import torch
        self.lib = load_library()
        self.cfg = cfg
        self.sizes = workspace_size(cfg)
        dev = torch.device(device)
        n = self.sizes["n_params"]
        if params is None:
            raise ValueError("initial params are the caller's (reading A-14)")
        self.params = torch.as_tensor(params, dtype=torch.float32).to(dev).contiguous().clone()
        assert self.params.numel() == n, (self.params.numel(), n)
        self.adam_m = torch.zeros(n, dtype=torch.float32, device=dev)
        self.adam_v = torch.zeros(n, dtype=torch.float32, device=dev)
        self.buffer = torch.empty(self.sizes["buffer_bytes"], dtype=torch.uint8, device=dev)
        self.scratch = torch.zeros(self.sizes["scratch_bytes"], dtype=torch.uint8, device=dev)
        na = self.sizes["n_actor_params"]
        self.actor_params = self.actor_m = self.actor_v = None
        if na:
            if actor_params is None:
                raise ValueError("actor params required when actor_depth > 0")
            self.actor_params = torch.as_tensor(actor_params, dtype=torch.float32).to(dev).contiguous().clone()
            self.actor_m = torch.zeros(na, dtype=torch.float32, device=dev)
            self.actor_v = torch.zeros(na, dtype=torch.float32, device=dev)
        mem = _Memory(params=self.params.data_ptr(), adam_m=self.adam_m.data_ptr(),
                      adam_v=self.adam_v.data_ptr(),
                      actor_params=self.actor_params.data_ptr() if na else None,
                      actor_adam_m=self.actor_m.data_ptr() if na else None,
                      actor_adam_v=self.actor_v.data_ptr() if na else None,
                      buffer=self.buffer.data_ptr(), scratch=self.scratch.data_ptr())
        idbuf = None
        if cfg.world_size > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("world_size > 1 needs the 128-byte NCCL unique id")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        torch.cuda.synchronize(dev)
        h = ctypes.c_void_p()
        _check(self.lib.crl_create(ctypes.byref(cfg._c()), ctypes.byref(mem), idbuf, ctypes.byref(h)))
        self._h = h
        self.n_params = n

    # ------------------------------------------------------------------ hot-path calls
    def buffer_insert(self, obs, act, done, stream=None):
        U = obs.shape[0]
        _check(self.lib.crl_buffer_insert(self._h, _ptr(obs), _ptr(act), _ptr(done), U,
                                          _stream(stream)), self._h)

    def relabel_sample(self, seed, step, s, a, g, idx=None, stream=None):
        _check(self.lib.crl_relabel_sample(self._h, seed, step, _ptr(s), _ptr(a), _ptr(g),
                                           _ptr(idx), _stream(stream)), self._h)

    def relabel_sample_bulk(self, seed, step0, n_updates, s, a, g, idx=None, stream=None):
        """n_updates batches in one launch: row u*B_l + r = row r of relabel_sample(seed, step0 + u)."""
        _check(self.lib.crl_relabel_sample_bulk(self._h, seed, step0, int(n_updates), _ptr(s), _ptr(a),
                                                _ptr(g), _ptr(idx), _stream(stream)), self._h)

    def relabel_sample_mixed(self, seed, step0, n_updates, s, a, g, g_actor, idx=None, stream=None):
        """As relabel_sample_bulk, plus the actor's goals with random-goal mixing in g_actor."""
        _check(self.lib.crl_relabel_sample_mixed(self._h, seed, step0, int(n_updates), _ptr(s), _ptr(a),
                                                 _ptr(g), _ptr(g_actor), _ptr(idx), _stream(stream)), self._h)

    def critic_step(self, s, a, g, loss_out=None, grads_out=None, stream=None):
        _check(self.lib.crl_critic_step(self._h, _ptr(s), _ptr(a), _ptr(g), _ptr(loss_out),
                                        _ptr(grads_out), _stream(stream)), self._h)

    def actor_loss(self, s, g, eps, alpha_ent, loss_out=None, actor_grads_out=None,
                   apply_adam=False, stream=None):
        _check(self.lib.crl_actor_loss(self._h, _ptr(s), _ptr(g), _ptr(eps), float(alpha_ent),
                                       _ptr(loss_out), _ptr(actor_grads_out), int(apply_adam),
                                       _stream(stream)), self._h)

    def entropy_update(self, log_alpha, target_entropy=None, lr=3e-4, alpha_out=None, loss_out=None,
                       stream=None):
        """One Adam step on the entropy coefficient (crl_entropy_update); log_alpha is a device
        float[1] updated in place.  Default target entropy -act_dim / 2 (reading A-32)."""
        if target_entropy is None:
            target_entropy = -0.5 * self.cfg.act_dim
        _check(self.lib.crl_entropy_update(self._h, float(target_entropy), float(lr), _ptr(log_alpha),
                                           _ptr(alpha_out), _ptr(loss_out), _stream(stream)), self._h)

    # ------------------------------------------------------------------ utilities
    def status(self, sync=True, reset=False) -> int:
        return self.lib.crl_get_status(self._h, int(sync), int(reset))

    def launch_count(self) -> int:
        return self.lib.crl_last_launch_count(self._h)

    def profile_enable(self, on: bool):
        _check(self.lib.crl_profile_enable(self._h, int(on)), self._h)

    def profile_read(self) -> dict:
        """{stage: (total_ms, launches)} accumulated since profile_enable."""
        n = self.lib.crl_profile_read(self._h, -1, None, 0, None, None)
        out = {}
        for i in range(n):
            name = ctypes.create_string_buffer(96)
            ms = ctypes.c_double(); cnt = ctypes.c_int()
            self.lib.crl_profile_read(self._h, i, name, 96, ctypes.byref(ms), ctypes.byref(cnt))
            out[name.value.decode()] = (ms.value, cnt.value)
        return out

    def debug_tensor(self, name):
        import torch
        p = ctypes.c_void_p(); n = ctypes.c_size_t()
        _check(self.lib.crl_debug_tensor(self._h, name.encode(), ctypes.byref(p), ctypes.byref(n)), self._h)
        torch.cuda.synchronize()
        # device -> device copy through torch: wrap the raw pointer with a cuda array interface
        return torch.as_tensor(_DevView(p.value, n.value), device=self.params.device).clone()

    def close(self):
        if getattr(self, "_h", None):
            self.lib.crl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DevView:
    """Minimal __cuda_array_interface__ over a raw fp32 device pointer (read-only view)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.crl_nccl_unique_id(buf))
    return buf.raw


def bootstrap_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it (plumbing)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
