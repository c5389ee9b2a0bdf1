"""Counter-based synthetic trajectory batches.

Every random number is ``splitmix64(mix(seed) ^ (array_id << 56) ^ index)`` where
``index`` is a GLOBAL coordinate (time step, global env column, feature), so a rank's
shard of columns is bit-identical to the same columns of the full batch: K shards
concatenate exactly to the K=1 batch.

Nothing here computes any part of the method (no GAE, normalisation, network or loss).
"""
from __future__ import annotations

import numpy as np

from .configs import Config

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# array ids (high byte of the counter key)
A_REW, A_REW2, A_DONE, A_VAL, A_OBS, A_ACT, A_XI, A_PHASE, A_PARAM = 1, 2, 3, 4, 5, 6, 7, 8, 9


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _seed_mix(seed: int) -> np.uint64:
    return splitmix64(np.array([seed], dtype=np.uint64))[0]


def uniform(seed: int, array_id: int, index) -> np.ndarray:
    """U[0,1) doubles for integer counter(s) ``index`` (53-bit mantissa)."""
    idx = np.asarray(index, dtype=np.uint64)
    key = idx ^ (np.uint64(array_id) << np.uint64(56)) ^ _seed_mix(seed)
    return (splitmix64(key) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, array_id: int, index) -> np.ndarray:
    """N(0,1) by Box-Muller on counters 2i and 2i+1 (cosine branch only)."""
    idx = np.asarray(index, dtype=np.uint64)
    u1 = uniform(seed, array_id, idx * np.uint64(2))
    u2 = uniform(seed, array_id, idx * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def shard_columns(cfg: Config, world: int, rank: int):
    """Contiguous block of env columns for ``rank`` (an env's agent columns stay together)."""
    n_env = cfg.B // cfg.agents
    if n_env % world:
        raise ValueError(f"{cfg.name}: {n_env} envs do not split over {world} ranks")
    e = n_env // world
    return rank * e * cfg.agents, (rank + 1) * e * cfg.agents


_VALUE_SIGMA = {"tiny": 10.0, "atari": 1.0, "gfootball": 1.0, "smac": 5.0, "hns": 1.0}


def _rewards_dones(cfg: Config, seed: int, c0: int, c1: int, stress: bool):
    T, Bg = cfg.T, cfg.B
    t = np.arange(T, dtype=np.uint64)[:, None]
    col = np.arange(c0, c1, dtype=np.uint64)[None, :]
    tc = t * np.uint64(Bg) + col                    # global (t, column) counter
    env = col // np.uint64(cfg.agents)
    n_env = np.uint64(Bg // cfg.agents)
    te = t * n_env + env                            # global (t, env) counter
    shape = (T, c1 - c0)
    rec = cfg.recipe
    if rec == "tiny":                               # CartPole-like +1 per step, Geometric(20) episodes
        r = np.ones(shape)
        d = uniform(seed, A_DONE, tc) < 1.0 / 20
    elif rec == "atari":                            # sparse +-1 (p=0.01 each), Geometric(800) episodes
        u = uniform(seed, A_REW, tc)
        r = np.where(u < 0.01, 1.0, np.where(u < 0.02, -1.0, 0.0))
        d = uniform(seed, A_DONE, tc) < 1.0 / 800
    elif rec == "gfootball":                        # goals +-1 (5e-4), +0.1 shaping (0.01); 3001-step episodes
        u = uniform(seed, A_REW, tc)
        sh = np.where(uniform(seed, A_REW2, tc) < 0.01, 0.1, 0.0)
        r = np.where(u < 5e-4, 1.0, np.where(u < 1e-3, -1.0, sh))
        phase = np.floor(uniform(seed, A_PHASE, col) * 3001).astype(np.int64)
        d = (t.astype(np.int64) + phase) % 3001 == 3000
    elif rec == "smac":                             # dense U(0,0.2) per env-step, +10 win at episode end
        dense = 0.2 * uniform(seed, A_REW, te)
        d = uniform(seed, A_DONE, te) < 1.0 / 120
        win = uniform(seed, A_REW2, te) < 0.5
        r = dense + np.where(d & win, 10.0, 0.0)
    elif rec == "hns":                              # 240-step episodes, 40% prep, +-1 team reward
        phase = np.floor(uniform(seed, A_PHASE, env) * 240).astype(np.int64)
        step = (t.astype(np.int64) + phase) % 240
        d = step == 239
        seen = uniform(seed, A_REW, te) < 0.5
        seeker = (col % np.uint64(cfg.agents)) >= np.uint64(cfg.agents // 2)
        r = np.where(seen == seeker, 1.0, -1.0)
        r = np.where(step < 96, 0.0, r)
    else:
        raise ValueError(rec)
    if stress:
        d = uniform(seed, A_DONE + 64, tc) < 0.1
    r = np.broadcast_to(r, shape)
    d = np.broadcast_to(d, shape)
    return np.ascontiguousarray(r, dtype=np.float32), np.ascontiguousarray(d, dtype=np.uint8)


def make_batch(cfg: Config, seed: int = 0, world: int = 1, rank: int = 0, *,
               stress: bool = False, with_obs: bool = True, ld_obs: int | None = None,
               chunk_rows: int = 1 << 16):
    """Rank ``rank``'s shard of one trajectory batch.

    Returns a dict of numpy arrays (time-major; local sample i = t * Bk + b):
      rewards f32 [T][Bk], values f32 [T+1][Bk] (row T = bootstrap), dones u8 [T][Bk],
      obs f16 [n][ld_obs] (pad columns zero), actions i32 [n][H], xi f64 [n] (the
      N(0, s^2) log-prob noise of the D-1 recipe; s = 0.15, 1.0 under ``stress``).
    """
    c0, c1 = shard_columns(cfg, world, rank)
    Bk, T, Bg = c1 - c0, cfg.T, cfg.B
    n = T * Bk
    rew, done = _rewards_dones(cfg, seed, c0, c1, stress)
    t1 = np.arange(T + 1, dtype=np.uint64)[:, None]
    col = np.arange(c0, c1, dtype=np.uint64)[None, :]
    val = (_VALUE_SIGMA[cfg.recipe] * normal(seed, A_VAL, t1 * np.uint64(Bg) + col)).astype(np.float32)

    # global sample counter of local sample i = t*Bk + b  ->  t*Bg + (c0 + b)
    tt = np.arange(T, dtype=np.uint64)[:, None]
    gs = (tt * np.uint64(Bg) + col).reshape(-1)           # [n]
    H = len(cfg.heads)
    act = np.empty((n, H), dtype=np.int32)
    for h, a in enumerate(cfg.heads):
        u = uniform(seed, A_ACT, gs * np.uint64(H) + np.uint64(h))
        act[:, h] = np.minimum(np.floor(u * a), a - 1).astype(np.int32)
    xi = (1.0 if stress else 0.15) * normal(seed, A_XI, gs)
    out = dict(rewards=rew, values=val, dones=done, actions=act, xi=xi,
               c0=c0, c1=c1, Bk=Bk, n=n)
    if with_obs:
        ld = cfg.ld_obs if ld_obs is None else ld_obs
        D = cfg.obs_dim
        obs = np.zeros((n, ld), dtype=np.float16)
        jj = np.arange(D, dtype=np.uint64)[None, :]
        for s in range(0, n, chunk_rows):
            g = gs[s:s + chunk_rows, None]
            z = normal(seed, A_OBS, g * np.uint64(D) + jj)
            obs[s:s + chunk_rows, :D] = np.clip(z, -5.0, 5.0).astype(np.float16)
        out["obs"] = obs
    return out


def logp_old_uniform_policy(cfg: Config, xi: np.ndarray) -> np.ndarray:
    """Behaviour log-prob for timing runs: a uniform policy per head, minus the noise xi."""
    return (-sum(np.log(a) for a in cfg.heads) - xi).astype(np.float32)


def make_params(cfg: Config, seed: int = 0, head_gain: float = 1.0) -> np.ndarray:
    """Flat f32 parameters in the SURVEY C-A10 layout: per layer W[out][in] then b[out].

    W, b ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in)) (PyTorch nn.Linear default, C-A11);
    the head layer is multiplied by ``head_gain``.
    """
    parts, off = [], 0
    for l, (fo, fi) in enumerate(cfg.layer_shapes):
        k = 1.0 / np.sqrt(fi)
        cnt = fo * fi + fo
        u = uniform(seed, A_PARAM, np.arange(off, off + cnt, dtype=np.uint64))
        p = (2.0 * u - 1.0) * k
        if l in cfg.head_layers:
            p = p * head_gain
        parts.append(p)
        off += cnt
    return np.concatenate(parts).astype(np.float32)
