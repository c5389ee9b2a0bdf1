"""ctypes binding of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2306_16688_b200``) never does; it shares no code with it.

``ppo_step`` composes the C functions in the order of one trainer step
(SURVEY.md §3.3): GAE per shard -> batch-wide normalisation over the union of the shards
-> loss and gradient per shard (scale 1/N_global, summed in rank order, C-5) -> Adam.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (no fast-math: IEEE double semantics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        # -fopenmp only for oracle_loss_and_grad_mt (bench.py's all-core timing); every
        # other function has no pragma and is the same single-threaded code
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-Wall", "-fopenmp",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32, u8 = C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_uint8)
        f = C.POINTER(C.c_float)
        ip = C.POINTER(C.c_int)
        _lib.oracle_gae.argtypes = [C.c_int, C.c_int, C.c_int, f, f, u8, f, C.c_double, C.c_double,
                                    d, d]
        _lib.oracle_moments.argtypes = [d, i64, d, d]
        _lib.oracle_adv_norm.argtypes = [d, i64, C.c_double, C.c_int, d, d, d]
        for sfx in ("", "_ac"):
            getattr(_lib, "oracle_param_count" + sfx).argtypes = [C.c_int, C.c_int, ip, C.c_int, ip]
            getattr(_lib, "oracle_param_count" + sfx).restype = i64
            getattr(_lib, "oracle_forward" + sfx).argtypes = [C.c_int, C.c_int, ip, C.c_int, ip, d, i64, d, d]
            getattr(_lib, "oracle_loss_and_grad" + sfx).argtypes = [
                C.c_int, C.c_int, ip, C.c_int, ip, d, i64, d, i32, d, d, d, C.c_double, C.c_double,
                C.c_double, C.c_double, d, d, d, d, C.c_double]
        _lib.oracle_loss_and_grad_mt.argtypes = [C.c_int, C.c_int, ip, C.c_int, ip, d, i64, d, i32,
                                                 d, d, d, C.c_double, C.c_double, C.c_double,
                                                 C.c_double, d, d, d, C.c_double, C.c_int, C.c_int]
        _lib.oracle_clip_grad_norm.argtypes = [i64, d, C.c_double]
        _lib.oracle_clip_grad_norm.restype = C.c_double
        u64 = C.POINTER(C.c_uint64)
        _lib.oracle_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        _lib.oracle_uniform.restype = C.c_double
        _lib.oracle_rollout.argtypes = [C.c_int, C.c_int, ip, C.c_int, ip, d, i64, d, u64,
                                        C.c_uint64, C.c_int, i32, d, d, d]
        _lib.oracle_adam.argtypes = [i64, d, d, d, d, i64, C.c_double, C.c_double, C.c_double,
                                     C.c_double]
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _ints(xs):
    arr = (C.c_int * max(1, len(xs)))(*xs)
    return arr


# ------------------------------------------------------------------ C-1
def gae(rewards, values, dones, gamma, lam, trunc_values=None):
    """rewards/dones [T][ld], values [T+1][ld] -> (adv, ret) float64 [T][B=ld].
    trunc_values [T][ld] (NEXT-3 R-T): flags with bit 1 set and bit 0 clear bootstrap from it."""
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    v = np.ascontiguousarray(values, dtype=np.float32)
    dd = np.ascontiguousarray(dones, dtype=np.uint8)
    T, ld = r.shape
    assert v.shape == (T + 1, ld) and dd.shape == (T, ld)
    tv = None if trunc_values is None else np.ascontiguousarray(trunc_values, dtype=np.float32)
    assert tv is None or tv.shape == (T, ld)
    adv = np.empty((T, ld), np.float64)
    ret = np.empty((T, ld), np.float64)
    lib().oracle_gae(T, ld, ld, _p(r, C.c_float), _p(v, C.c_float), _p(dd, C.c_uint8),
                     _p(tv, C.c_float) if tv is not None else None,
                     gamma, lam, _p(adv, C.c_double), _p(ret, C.c_double))
    return adv, ret


# ------------------------------------------------------------------ C-2
def moments(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    mu, m2 = C.c_double(), C.c_double()
    lib().oracle_moments(_p(a, C.c_double), a.size, C.byref(mu), C.byref(m2))
    return mu.value, m2.value


def adv_norm(a, eps=1e-8, unbiased=False):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    out = np.empty_like(a)
    mu, sd = C.c_double(), C.c_double()
    lib().oracle_adv_norm(_p(a, C.c_double), a.size, eps, int(unbiased), _p(out, C.c_double),
                          C.byref(mu), C.byref(sd))
    return out, mu.value, sd.value


# ------------------------------------------------------------------ C-3 / C-4
def _sfx(separate):
    return "_ac" if separate else ""


def param_count(obs_dim, hidden, heads, separate=False):
    """separate: the NEXT-3 separate actor / critic trunks (oracle_*_ac, reading R-AC)."""
    return getattr(lib(), "oracle_param_count" + _sfx(separate))(
        obs_dim, len(hidden), _ints(hidden), len(heads), _ints(heads))


def forward(obs_dim, hidden, heads, params, obs, separate=False):
    p = np.ascontiguousarray(params, dtype=np.float64)
    x = np.ascontiguousarray(obs, dtype=np.float64)[:, :obs_dim].copy()
    n = x.shape[0]
    out = np.empty((n, sum(heads) + 1), np.float64)
    getattr(lib(), "oracle_forward" + _sfx(separate))(
        obs_dim, len(hidden), _ints(hidden), len(heads), _ints(heads), _p(p, C.c_double), n,
        _p(x, C.c_double), _p(out, C.c_double))
    return out


def loss_and_grad(obs_dim, hidden, heads, params, obs, actions, logp_old, adv_hat, ret,
                  clip_eps=0.2, value_coef=0.5, entropy_coef=0.01, grad_scale=None,
                  grad=None, sums=None, want_per_sample=False, v_old=None, value_clip=0.0,
                  threads=1, separate=False):
    """threads > 1: the all-core timing driver (oracle_loss_and_grad_mt, block-order sums).
    separate: the separate actor / critic trunks (oracle_loss_and_grad_ac)."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    x = np.ascontiguousarray(np.asarray(obs, dtype=np.float64)[:, :obs_dim])
    n = x.shape[0]
    act = np.ascontiguousarray(actions, dtype=np.int32).reshape(n, len(heads))
    lo = np.ascontiguousarray(logp_old, dtype=np.float64).reshape(-1)
    ah = np.ascontiguousarray(adv_hat, dtype=np.float64).reshape(-1)
    rt = np.ascontiguousarray(ret, dtype=np.float64).reshape(-1)
    if grad is None:
        grad = np.zeros(p.size, np.float64)
    if sums is None:
        sums = np.zeros(5, np.float64)
    if grad_scale is None:
        grad_scale = 1.0 / n
    ps = np.empty(n, np.float64) if want_per_sample else None
    vo = None if v_old is None else np.ascontiguousarray(v_old, dtype=np.float64).reshape(-1)
    if threads > 1:
        assert not want_per_sample
        lib().oracle_loss_and_grad_mt(obs_dim, len(hidden), _ints(hidden), len(heads), _ints(heads),
                                      _p(p, C.c_double), n, _p(x, C.c_double), _p(act, C.c_int32),
                                      _p(lo, C.c_double), _p(ah, C.c_double), _p(rt, C.c_double),
                                      clip_eps, value_coef, entropy_coef, grad_scale,
                                      _p(grad, C.c_double), _p(sums, C.c_double),
                                      _p(vo, C.c_double) if vo is not None else None,
                                      float(value_clip), int(threads), int(bool(separate)))
        return grad, sums, None
    getattr(lib(), "oracle_loss_and_grad" + _sfx(separate))(obs_dim, len(hidden), _ints(hidden), len(heads), _ints(heads),
                               _p(p, C.c_double), n, _p(x, C.c_double), _p(act, C.c_int32),
                               _p(lo, C.c_double), _p(ah, C.c_double), _p(rt, C.c_double),
                               clip_eps, value_coef, entropy_coef, grad_scale,
                               _p(grad, C.c_double), _p(sums, C.c_double),
                               _p(ps, C.c_double) if ps is not None else None,
                               _p(vo, C.c_double) if vo is not None else None, float(value_clip))
    return grad, sums, ps


# ------------------------------------------------------------------ NEXT-3
def clip_grad_norm(g, max_norm):
    """In place on a float64 contiguous array; returns the pre-clip global norm."""
    assert g.dtype == np.float64 and g.flags.c_contiguous
    return lib().oracle_clip_grad_norm(g.size, _p(g, C.c_double), float(max_norm))


# ------------------------------------------------------------------ NEXT-2
def uniform(seed, key, h):
    return lib().oracle_uniform(int(seed), int(key), int(h))


def rollout(obs_dim, hidden, heads, params, obs, seed=0, keys=None, deterministic=False):
    """Policy-worker inference: (actions i32 [n][H], logp [n], value [n], margin [n][H])."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    x = np.ascontiguousarray(np.asarray(obs, dtype=np.float64)[:, :obs_dim])
    n = x.shape[0]
    H = len(heads)
    k = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint64)
    act = np.empty((n, H), np.int32)
    lp, val, mg = np.empty(n), np.empty(n), np.empty((n, H))
    lib().oracle_rollout(obs_dim, len(hidden), _ints(hidden), H, _ints(heads), _p(p, C.c_double),
                         n, _p(x, C.c_double), _p(k, C.c_uint64) if k is not None else None,
                         int(seed), int(bool(deterministic)), _p(act, C.c_int32),
                         _p(lp, C.c_double), _p(val, C.c_double), _p(mg, C.c_double))
    return act, lp, val, mg


# ------------------------------------------------------------------ C-6
def adam(p, m, v, g, t, lr=3e-4, b1=0.9, b2=0.999, eps=1e-8):
    """In place on float64 contiguous arrays."""
    for a in (p, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = np.ascontiguousarray(g, dtype=np.float64)
    lib().oracle_adam(p.size, _p(p, C.c_double), _p(m, C.c_double), _p(v, C.c_double),
                      _p(g, C.c_double), int(t), lr, b1, b2, eps)


# ------------------------------------------------------------------ one trainer step
def log_pi(cfg, params, obs, actions):
    """log pi_theta(a|s) summed over heads, by the oracle forward (test-fixture helper)."""
    z = forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, obs, separate=sep(cfg))
    out = np.zeros(z.shape[0])
    s = 0
    for h, a in enumerate(cfg.heads):
        zz = z[:, s:s + a]
        mx = zz.max(axis=1, keepdims=True)
        lsm = zz - (mx + np.log(np.exp(zz - mx).sum(axis=1, keepdims=True)))
        out += lsm[np.arange(z.shape[0]), actions[:, h]]
        s += a
    return out


def sep(cfg):
    return bool(getattr(cfg, "separate_critic", False))


def minibatch_bounds(n, M):
    """NEXT-3 reading R-M: local minibatch k of M covers sample rows [k*n//M, (k+1)*n//M)
    of the time-major flattened shard (contiguous, no shuffle)."""
    return [(k * n // M, (k + 1) * n // M) for k in range(M)]


def default_threads():
    """Threads of the oracle's block driver in ppo_step (ORACLE_THREADS, default all cores)."""
    try:
        return max(1, int(os.environ.get("ORACLE_THREADS", "0")) or len(os.sched_getaffinity(0)))
    except Exception:
        return 1


def ppo_step(cfg, params, shards, *, eps=1e-8, unbiased=False, adam_state=None, t=1,
             apply=True, value_clip=0.0, max_grad_norm=0.0, epochs=1, minibatches=1, threads=None):
    """One trainer step of the oracle over K shards (list of dicts from synth.make_batch
    with a ``logp_old`` entry).  Returns a dict with adv/ret per shard, mean/std, grad,
    loss sums and (if apply) the updated params/m/v.

    NEXT-3: value_clip > 0 clips the value loss around v_old = the
    rollout values (rows 0..T-1 of each shard's ``values``); max_grad_norm > 0 clips the
    global gradient (after the rank-order sum, before Adam); epochs x minibatches runs
    E*M Adam updates, minibatch k being the union over ranks of each shard's local rows
    ``minibatch_bounds(n_local, M)[k]``.  Normalisation statistics are taken once over the
    whole batch.  With E*M > 1 the per-update gradients are returned in ``grads`` and
    ``grad``/``sums`` are those of the last update.

    Optional shard keys (NEXT-3): ``trunc_values`` [T][Bk] (reading R-T, time-limit
    bootstrap in GAE) and ``valid`` [T][Bk] u8 (reading R-P: padding samples, valid = 0,
    are left out of the normalisation moments, the loss and N).

    threads: the per-sample loss/gradient of a shard with >= 1024 rows goes through the
    block driver (oracle_loss_and_grad_mt: the same per-sample arithmetic, block sums added in
    block order -- pinned to the 1-thread call); None = default_threads()."""
    if threads is None:
        threads = default_threads()
    advs, rets, vms = [], [], []
    for sh in shards:
        a, r = gae(sh["rewards"], sh["values"], sh["dones"], cfg.gamma, cfg.lam,
                   trunc_values=sh.get("trunc_values"))
        advs.append(a.reshape(-1))
        rets.append(r.reshape(-1))
        vm = sh.get("valid")
        vms.append(np.ones(a.size, bool) if vm is None else np.asarray(vm).reshape(-1) != 0)
    allA = np.concatenate([a[vm] for a, vm in zip(advs, vms)])
    N = allA.size
    _, mu, sd = adv_norm(allA, eps=eps, unbiased=unbiased)
    p64 = np.asarray(params, dtype=np.float64).copy()
    if adam_state is None:
        adam_state = (np.zeros_like(p64), np.zeros_like(p64))
    m, v = adam_state
    vold = [np.asarray(sh["values"], np.float64)[:-1].reshape(-1) for sh in shards]
    out = dict(adv=advs, ret=rets, mean=mu, std=sd, N=N, grads=[], norms=[], sums_all=[])
    for _ in range(epochs):
        for k in range(minibatches):
            grad = np.zeros(p64.size)
            sums = np.zeros(5)
            parts = []
            for sh, a, r, vo, vm in zip(shards, advs, rets, vold, vms):
                lo, hi = minibatch_bounds(a.size, minibatches)[k]
                rows = lo + np.nonzero(vm[lo:hi])[0]      # the valid rows of the range
                parts.append((sh, a, r, vo, rows))
            Nmb = sum(rows.size for *_, rows in parts)
            for sh, a, r, vo, rows in parts:               # rank order (C-5)
                if rows.size == 0:
                    continue
                ahat = (a[rows] - mu) / (sd + eps)
                loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, p64,
                              np.asarray(sh["obs"])[rows], np.asarray(sh["actions"])[rows],
                              np.asarray(sh["logp_old"])[rows], ahat, r[rows],
                              cfg.clip_eps, cfg.value_coef, cfg.entropy_coef,
                              grad_scale=1.0 / Nmb, grad=grad, sums=sums,
                              v_old=vo[rows] if value_clip > 0 else None,
                              value_clip=value_clip, threads=threads if rows.size >= 1024 else 1,
                              separate=sep(cfg))
            norm = clip_grad_norm(grad, max_grad_norm) if max_grad_norm > 0 else float(
                np.sqrt(np.sum(grad * grad)))
            out["grads"].append(grad)
            out["norms"].append(norm)
            out["sums_all"].append(sums)
            if apply:
                adam(p64, m, v, grad, t, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
                t += 1
    out.update(grad=grad, sums=sums, grad_norm=out["norms"][-1])
    if apply:
        out.update(params=p64, m=m, v=v)
    return out
