"""Thin ctypes binding of libsrl.so (include/srl.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  torch supplies device memory, streams
and process groups.  There is no CPU fallback: a missing or unloadable library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# SRL_LIB: load another build of the same library (tools/build_variant.py experiments)
SO = os.environ.get("SRL_LIB") or os.path.join(HERE, "libsrl.so")

SRL_OK, SRL_EINVAL, SRL_ECUDA, SRL_ENCCL, SRL_ENOMEM, SRL_EUNSUPPORTED, SRL_ESTATE = range(7)

# every symbol include/srl.h declares (checked by tests/test_abi.py)
EXPORTS = ("srl_last_error", "srl_abi_version", "srl_gae", "srl_adv_norm", "srl_nccl_unique_id",
           "srl_ppo_create", "srl_ppo_destroy", "srl_ppo_params", "srl_ppo_adam_state",
           "srl_ppo_load_params", "srl_ppo_step", "srl_ppo_train_step", "srl_batch_upload",
           "srl_ppo_train_step_slot", "srl_policy_rollout", "srl_ppo_comm_path",
           "srl_allreduce_grads", "srl_prof_enable",
           "srl_prof_reset", "srl_prof_count", "srl_prof_read", "srl_debug_gemm",
           "srl_debug_exchange")


class SrlError(RuntimeError):
    pass


class PPOConfigC(C.Structure):
    _fields_ = [("obs_dim", C.c_int), ("ld_obs", C.c_int), ("n_hidden", C.c_int),
                ("hidden", C.POINTER(C.c_int)), ("n_heads", C.c_int),
                ("head_sizes", C.POINTER(C.c_int)),
                ("clip_eps", C.c_float), ("value_coef", C.c_float), ("entropy_coef", C.c_float),
                ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("adam_eps", C.c_float), ("adv_eps", C.c_float),
                ("gamma", C.c_float), ("gae_lambda", C.c_float), ("adv_unbiased", C.c_int),
                ("max_local_n", C.c_int64), ("precision", C.c_int),
                # NEXT-3 PPO variants
                ("value_clip", C.c_float), ("max_grad_norm", C.c_float),
                ("epochs", C.c_int), ("minibatches", C.c_int), ("separate_critic", C.c_int)]


class PPOStatsC(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("policy_loss", "value_loss", "entropy", "clip_fraction",
                                          "approx_kl", "loss", "adv_mean", "adv_std")] + \
               [(k, C.c_int64) for k in ("n_global", "nonfinite", "fp16_saturated", "step")] + \
               [("grad_norm", C.c_double), ("comm_error", C.c_int64)]


STATS_BYTES = C.sizeof(PPOStatsC)
STATS_FIELDS = [f for f, _ in PPOStatsC._fields_]

_lib = None


def lib():
    """Load libsrl.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        raise SrlError(f"{SO} is missing: run `python -m paper_2306_16688_b200.build` "
                       "(there is no CPU fallback)")
    L = C.CDLL(SO)
    vp, i64, st = C.c_void_p, C.c_int64, C.c_int
    L.srl_last_error.restype = C.c_char_p
    L.srl_abi_version.restype = C.c_int
    L.srl_gae.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_float, C.c_float,
                          vp, vp, vp, vp]
    L.srl_adv_norm.argtypes = [vp, vp, i64, vp, C.c_float, C.c_int, C.c_int, vp, vp]
    L.srl_nccl_unique_id.argtypes = [C.c_char_p]
    L.srl_ppo_create.argtypes = [C.POINTER(PPOConfigC), C.c_int, C.c_int, C.c_char_p, C.c_int,
                                 C.POINTER(vp)]
    L.srl_ppo_destroy.argtypes = [vp]
    L.srl_ppo_params.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64), C.POINTER(C.c_uint64)]
    L.srl_ppo_adam_state.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)]
    L.srl_ppo_load_params.argtypes = [vp, vp, vp]
    L.srl_ppo_step.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp]
    L.srl_ppo_train_step.argtypes = [vp, C.c_int, C.c_int, i64, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp, vp]
    L.srl_batch_upload.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp]
    L.srl_ppo_train_step_slot.argtypes = [vp, C.c_int, i64, vp, vp]
    L.srl_ppo_comm_path.argtypes = [vp]
    L.srl_ppo_comm_path.restype = C.c_int
    L.srl_policy_rollout.argtypes = [vp, i64, vp, vp, C.c_uint64, C.c_int, vp, vp, vp, vp]
    L.srl_allreduce_grads.argtypes = [vp, vp, i64, C.c_int, vp]
    L.srl_debug_gemm.argtypes = [C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.c_int,
                                 C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
    L.srl_debug_exchange.argtypes = [C.c_int, i64, i64, vp, vp, C.c_float, vp, vp, C.c_int, vp]
    L.srl_prof_enable.argtypes = [vp, C.c_int]
    L.srl_prof_reset.argtypes = [vp]
    L.srl_prof_count.argtypes = [vp]
    L.srl_prof_read.argtypes = [vp, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_float),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]
    for name in EXPORTS[2:]:
        getattr(L, name).restype = st
    _lib = L
    return L


def _check(rc):
    if rc != SRL_OK:
        raise SrlError(f"libsrl status {rc}: {lib().srl_last_error().decode()}")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _cuda(t, dtype, name, shape=None, numel=None):
    """Argument check before the C call (the library trusts shapes it cannot see)."""
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise SrlError(f"{name}: need a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise SrlError(f"{name}: need shape {tuple(shape)}, got {tuple(t.shape)}")
    if numel is not None and t.numel() != numel:
        raise SrlError(f"{name}: need {numel} elements, got {t.numel()}")
    return t


def _host(t, dtype, name, numel):
    if t.is_cuda or t.dtype != dtype or not t.is_contiguous() or t.numel() != numel:
        raise SrlError(f"{name}: need a contiguous host {dtype} tensor of {numel} elements, got "
                       f"{t.dtype} {tuple(t.shape)} on {t.device}")
    return t


# ------------------------------------------------------------------ a1
def gae(rewards, values, dones, gamma, lam, adv=None, ret=None, stats=None, ld=None, stream=None,
        trunc_values=None, valid=None):
    """srl_gae on [T][ld] tensors; returns (adv, ret, stats{n, mean, M2} f64[3])."""
    _cuda(rewards, torch.float32, "rewards")
    _cuda(values, torch.float32, "values")
    _cuda(dones, torch.uint8, "dones")
    if trunc_values is not None:
        _cuda(trunc_values, torch.float32, "trunc_values")
    if valid is not None:
        _cuda(valid, torch.uint8, "valid")
    T, ldr = rewards.shape
    B = ldr if ld is None else ld
    if adv is None:
        adv = torch.empty_like(rewards)
    if ret is None:
        ret = torch.empty_like(rewards)
    if stats is None:
        stats = torch.empty(3, dtype=torch.float64, device=rewards.device)
    _check(lib().srl_gae(T, B, ldr, _ptr(rewards), _ptr(values), _ptr(dones), _ptr(trunc_values),
                         _ptr(valid), gamma, lam,
                         _ptr(adv), _ptr(ret), _ptr(stats), _stream(stream)))
    return adv, ret, stats


# ------------------------------------------------------------------ a2
def adv_norm(adv, local_stats=None, eps=1e-8, unbiased=False, apply=False, ctx=None,
             mean_std=None, stream=None):
    _cuda(adv, torch.float32, "adv")
    if mean_std is None:
        mean_std = torch.empty(2, dtype=torch.float64, device=adv.device)
    h = ctx.handle if ctx is not None else None
    _check(lib().srl_adv_norm(h, _ptr(adv), adv.numel(), _ptr(local_stats), eps, int(unbiased),
                              int(apply), _ptr(mean_std), _stream(stream)))
    return mean_std


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().srl_nccl_unique_id(buf))
    return buf.raw


def _cudart():
    lib()
    return C.CDLL("libcudart.so.12")


def copy_from_device_ptr(dst: torch.Tensor, src_ptr: int, nbytes: int, stream=None):
    """cudaMemcpyAsync(dst <- raw device pointer), stream-ordered."""
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    rc = rt.cudaMemcpyAsync(C.c_void_p(dst.data_ptr()), C.c_void_p(src_ptr), nbytes, 3,
                            _stream(stream))
    if rc != 0:
        raise SrlError(f"cudaMemcpyAsync failed: {rc}")
    return dst


@dataclass
class NetSpec:
    obs_dim: int
    hidden: tuple
    heads: tuple
    ld_obs: int = 0
    clip_eps: float = 0.2
    value_coef: float = 0.5
    entropy_coef: float = 0.01
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    adv_eps: float = 1e-8
    gamma: float = 0.99
    gae_lambda: float = 0.95
    adv_unbiased: int = 0
    value_clip: float = 0.0       # NEXT-3
    max_grad_norm: float = 0.0
    epochs: int = 1
    minibatches: int = 1
    separate_critic: int = 0      # NEXT-3 R-AC

    @classmethod
    def from_config(cls, cfg):
        return cls(cfg.obs_dim, tuple(cfg.hidden), tuple(cfg.heads), cfg.ld_obs, cfg.clip_eps,
                   cfg.value_coef, cfg.entropy_coef, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps,
                   1e-8, cfg.gamma, cfg.lam, 0,
                   separate_critic=int(bool(getattr(cfg, "separate_critic", False))))


class PPOContext:
    """Owns an srl_ctx: params (f32 master + f16 shadows), Adam state, gradient bucket,
    workspace and (world > 1) the NCCL communicator."""

    def __init__(self, spec: NetSpec, max_local_n: int, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, device: int | None = None):
        self.spec = spec
        self.device = torch.cuda.current_device() if device is None else device
        self._hid = (C.c_int * len(spec.hidden))(*spec.hidden)
        self._heads = (C.c_int * len(spec.heads))(*spec.heads)
        ld = spec.ld_obs or (spec.obs_dim + 7) // 8 * 8
        self.ld_obs = ld
        self.cfg = PPOConfigC(spec.obs_dim, ld, len(spec.hidden), self._hid, len(spec.heads),
                              self._heads, spec.clip_eps, spec.value_coef, spec.entropy_coef,
                              spec.lr, spec.beta1, spec.beta2, spec.adam_eps, spec.adv_eps,
                              spec.gamma, spec.gae_lambda, int(spec.adv_unbiased),
                              int(max_local_n), 0, spec.value_clip, spec.max_grad_norm,
                              int(spec.epochs), int(spec.minibatches), int(spec.separate_critic))
        h = C.c_void_p()
        _check(lib().srl_ppo_create(C.byref(self.cfg), rank, world, nccl_id, self.device,
                                    C.byref(h)))
        self.handle = h
        self.rank, self.world = rank, world
        p, g, P, dg = C.c_void_p(), C.c_void_p(), C.c_int64(), C.c_uint64()
        _check(lib().srl_ppo_params(h, C.byref(p), C.byref(g), C.byref(P), C.byref(dg)))
        self.params_ptr, self.grads_ptr, self.P, self.layout_digest = p.value, g.value, P.value, dg.value
        m, v, t = C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(lib().srl_ppo_adam_state(h, C.byref(m), C.byref(v), C.byref(t)))
        self.m_ptr, self.v_ptr = m.value, v.value

    def close(self):
        if getattr(self, "handle", None):
            lib().srl_ppo_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_params(self, params: torch.Tensor, stream=None):
        _cuda(params, torch.float32, "params")
        assert params.numel() == self.P
        _check(lib().srl_ppo_load_params(self.handle, _ptr(params), _stream(stream)))

    def _read(self, ptr, n, stream=None):
        out = torch.empty(n, dtype=torch.float32, device=f"cuda:{self.device}")
        return copy_from_device_ptr(out, ptr, 4 * n, stream)

    def params(self, stream=None):
        return self._read(self.params_ptr, self.P, stream)

    def grads(self, stream=None):
        """The gradient bucket [P + 8] (gradients, then the 8 reduced statistics)."""
        return self._read(self.grads_ptr, self.P + 8, stream)

    def adam_state(self, stream=None):
        return self._read(self.m_ptr, self.P, stream), self._read(self.v_ptr, self.P, stream)

    def step(self, n_global, obs, actions, logp_old, adv, ret, adv_mean_std=None, apply=True,
             stats=None, stream=None, v_old=None, valid=None):
        """srl_ppo_step; returns the device stats buffer (uint8 [sizeof srl_ppo_stats])."""
        n_local = logp_old.numel()
        H, ld = len(self.spec.heads), self.ld_obs
        _cuda(obs, torch.float16, "obs", numel=n_local * ld)
        _cuda(actions, torch.int32, "actions", numel=n_local * H)
        for t, nm in ((logp_old, "logp_old"), (adv, "adv"), (ret, "ret")):
            _cuda(t, torch.float32, nm, numel=n_local)
        if v_old is not None:
            _cuda(v_old, torch.float32, "v_old", numel=n_local)
        if valid is not None:
            _cuda(valid, torch.uint8, "valid", numel=n_local)
        if stats is None:
            stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=obs.device)   # fully written
        _check(lib().srl_ppo_step(self.handle, n_local, int(n_global), _ptr(obs), _ptr(actions),
                                  _ptr(logp_old), _ptr(adv), _ptr(ret), _ptr(v_old), _ptr(valid),
                                  _ptr(adv_mean_std),
                                  int(apply), _ptr(stats), _stream(stream)))
        return stats

    def profile(self, on: bool = True):
        _check(lib().srl_prof_enable(self.handle, int(on)))

    def prof_reset(self):
        _check(lib().srl_prof_reset(self.handle))

    def prof_records(self):
        """[(name, ms, flops, bytes)] for every launch recorded since the last reset."""
        out = []
        nm, ms, fl, by = C.c_char_p(), C.c_float(), C.c_double(), C.c_double()
        for i in range(lib().srl_prof_count(self.handle)):
            _check(lib().srl_prof_read(self.handle, i, C.byref(nm), C.byref(ms), C.byref(fl),
                                       C.byref(by)))
            out.append((nm.value.decode(), ms.value, fl.value, by.value))
        return out

    def train_step(self, n_global, rewards, values, dones, obs, actions, logp_old, stats=None,
                   stream=None, trunc_values=None, valid=None):
        """srl_ppo_train_step: GAE -> normalisation -> update in one call (device inputs)."""
        T, B = rewards.shape
        n, H, ld = T * B, len(self.spec.heads), self.ld_obs
        _cuda(rewards, torch.float32, "rewards")
        _cuda(values, torch.float32, "values", shape=(T + 1, B))
        _cuda(dones, torch.uint8, "dones", shape=(T, B))
        _cuda(obs, torch.float16, "obs", numel=n * ld)
        _cuda(actions, torch.int32, "actions", numel=n * H)
        _cuda(logp_old, torch.float32, "logp_old", numel=n)
        if trunc_values is not None:
            _cuda(trunc_values, torch.float32, "trunc_values", shape=(T, B))
        if valid is not None:
            _cuda(valid, torch.uint8, "valid", numel=n)
        if stats is None:
            stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=obs.device)   # fully written
        _check(lib().srl_ppo_train_step(self.handle, T, B, int(n_global), _ptr(rewards),
                                        _ptr(values), _ptr(dones), _ptr(trunc_values),
                                        _ptr(valid), _ptr(obs), _ptr(actions),
                                        _ptr(logp_old), _ptr(stats), _stream(stream)))
        return stats

    def upload(self, slot, rewards, values, dones, obs, actions, logp_old, trunc_values=None,
               valid=None):
        """NEXT-1: async H2D of a host batch (pinned CPU tensors) into device slot 0/1."""
        T, B = rewards.shape
        n, H, ld = T * B, len(self.spec.heads), self.ld_obs
        _host(rewards, torch.float32, "rewards", n)
        _host(values, torch.float32, "values", (T + 1) * B)
        _host(dones, torch.uint8, "dones", n)
        _host(obs, torch.float16, "obs", n * ld)
        _host(actions, torch.int32, "actions", n * H)
        _host(logp_old, torch.float32, "logp_old", n)
        if trunc_values is not None:
            _host(trunc_values, torch.float32, "trunc_values", n)
        if valid is not None:
            _host(valid, torch.uint8, "valid", n)
        _check(lib().srl_batch_upload(self.handle, slot, T, B, _ptr(rewards), _ptr(values),
                                      _ptr(dones), _ptr(obs), _ptr(actions), _ptr(logp_old),
                                      _ptr(trunc_values), _ptr(valid)))

    def train_step_slot(self, slot, n_global, stats=None, stream=None):
        if stats is None:
            stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=f"cuda:{self.device}")   # fully written
        _check(lib().srl_ppo_train_step_slot(self.handle, slot, int(n_global), _ptr(stats),
                                             _stream(stream)))
        return stats

    def rollout(self, obs, keys=None, seed=0, deterministic=False, actions=None, logp=None,
                value=None, stream=None):
        """NEXT-2 srl_policy_rollout: batched policy inference -> (actions i32 [n][H], logp, value)."""
        n = obs.shape[0]
        _cuda(obs, torch.float16, "obs", numel=n * self.ld_obs)
        if keys is not None:
            _cuda(keys, torch.int64, "keys", numel=n)
        dev = obs.device
        if actions is None:
            actions = torch.empty((n, len(self.spec.heads)), dtype=torch.int32, device=dev)
        if logp is None:
            logp = torch.empty(n, dtype=torch.float32, device=dev)
        if value is None:
            value = torch.empty(n, dtype=torch.float32, device=dev)
        _check(lib().srl_policy_rollout(self.handle, n, _ptr(obs), _ptr(keys), int(seed) & ((1 << 64) - 1),
                                        int(bool(deterministic)), _ptr(actions), _ptr(logp),
                                        _ptr(value), _stream(stream)))
        return actions, logp, value

    @property
    def comm_path(self) -> str:
        """a6 path of srl_ppo_step: 'none' (world 1), 'nccl' or 'nvlink-p2p'."""
        return {0: "none", 1: "nccl", 2: "nvlink-p2p"}[lib().srl_ppo_comm_path(self.handle)]

    def allreduce_grads(self, buf: torch.Tensor, op: int = 0, stream=None):
        _cuda(buf, torch.float32, "buf")
        _check(lib().srl_allreduce_grads(self.handle, _ptr(buf), buf.numel(), op, _stream(stream)))
        return buf


def decode_stats(stats_u8: torch.Tensor) -> dict:
    raw = bytes(stats_u8.cpu().numpy().tobytes())
    s = PPOStatsC.from_buffer_copy(raw)
    return {k: getattr(s, k) for k in STATS_FIELDS}


def debug_gemm(A, a_mn, B, b_mn, M, N, K, bn=128, splits=1, cg=1, stream=None):
    """Test hook: D[M][N] = sum_k A(m,k) B(n,k) through the tcgen05 GEMM (EPI_PART path)."""
    D = torch.empty(M, N, dtype=torch.float32, device=A.device)
    _check(lib().srl_debug_gemm(M, N, K, _ptr(A), int(a_mn), A.shape[1], _ptr(B), int(b_mn),
                                B.shape[1], bn, splits, cg, _ptr(D), _stream(stream)))
    return D


def debug_exchange(x, scale=1.0, tri=None, unbiased=False, stream=None):
    """Test hook (srl_debug_exchange): the a6/a2 peer-memory exchange kernels for
    world = x.shape[0] virtual ranks on this GPU.  x f32 [world][ld] (reduced in place);
    returns (out [world][ld], mean_std [world][2] or None)."""
    _cuda(x, torch.float32, "x")
    world, ld = x.shape
    out = torch.zeros_like(x)
    ms = None
    if tri is not None:
        _cuda(tri, torch.float64, "tri", shape=(world, 3))
        ms = torch.zeros((world, 2), dtype=torch.float64, device=x.device)
    count = ld
    _check(lib().srl_debug_exchange(world, count, ld, _ptr(x), _ptr(out), float(scale), _ptr(tri),
                                    _ptr(ms), int(unbiased), _stream(stream)))
    return out, ms
