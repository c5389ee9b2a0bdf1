"""Device-side synthetic batches for TIMING runs of the large configs (SMAC, HnS), where the
host counter generator (gen.py) would take minutes.  Same shapes, dtypes and reward / done /
value / observation / action distributions as gen.py's D-1 recipe, drawn
with torch's device RNG instead of the counter stream, so the arrays are NOT bit-identical
to gen.py's: they are timing inputs only, never parity inputs.

Like gen.py, nothing here computes any part of the method.
"""
from __future__ import annotations

import math

import torch

from .configs import Config

_VALUE_SIGMA = {"tiny": 10.0, "atari": 1.0, "gfootball": 1.0, "smac": 5.0, "hns": 1.0}


def make_batch_device(cfg: Config, device, seed: int = 0, world: int = 1, rank: int = 0):
    """This rank's shard (B / world columns) as device tensors: rewards f32 [T][Bk], values
    f32 [T+1][Bk], dones u8 [T][Bk], obs f16 [n][ld_obs], actions i32 [n][H], logp_old f32 [n]
    (uniform behaviour policy minus N(0, 0.15^2) noise, the bench recipe)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1009 + rank)
    T = cfg.T
    n_env = cfg.B // cfg.agents
    if n_env % world:
        raise ValueError(f"{cfg.name}: {n_env} envs do not split over {world} ranks")
    Ek = n_env // world
    Bk = Ek * cfg.agents
    n = T * Bk
    A = cfg.agents
    U = lambda *s: torch.rand(*s, generator=g, device=device, dtype=torch.float32)
    rec = cfg.recipe
    t = torch.arange(T, device=device)[:, None]
    if rec == "tiny":
        r = torch.ones(T, Bk, device=device)
        d = U(T, Bk) < 1.0 / 20
    elif rec == "atari":
        u = U(T, Bk)
        r = torch.where(u < 0.01, 1.0, torch.where(u < 0.02, -1.0, 0.0))
        d = U(T, Bk) < 1.0 / 800
    elif rec == "gfootball":
        u = U(T, Bk)
        sh = torch.where(U(T, Bk) < 0.01, 0.1, 0.0)
        r = torch.where(u < 5e-4, 1.0, torch.where(u < 1e-3, -1.0, sh))
        phase = torch.floor(U(1, Bk) * 3001).long()
        d = (t + phase) % 3001 == 3000
    elif rec == "smac":
        dense = 0.2 * U(T, Ek)
        de = U(T, Ek) < 1.0 / 120
        win = U(T, Ek) < 0.5
        r = (dense + torch.where(de & win, 10.0, 0.0)).repeat_interleave(A, dim=1)
        d = de.repeat_interleave(A, dim=1)
    elif rec == "hns":
        phase = torch.floor(U(1, Ek) * 240).long().repeat_interleave(A, dim=1)
        step = (t + phase) % 240
        d = step == 239
        seen = (U(T, Ek) < 0.5).repeat_interleave(A, dim=1)
        seeker = (torch.arange(Bk, device=device) % A >= A // 2)[None, :]
        r = torch.where(seen == seeker, 1.0, -1.0)
        r = torch.where(step < 96, 0.0, r)
    else:
        raise ValueError(rec)
    values = _VALUE_SIGMA[rec] * torch.randn(T + 1, Bk, generator=g, device=device)
    obs = torch.zeros(n, cfg.ld_obs, dtype=torch.float16, device=device)
    rows = 1 << 20
    for s in range(0, n, rows):
        e = min(n, s + rows)
        obs[s:e, :cfg.obs_dim] = torch.randn(e - s, cfg.obs_dim, generator=g, device=device).clamp_(-5, 5).half()
    H = len(cfg.heads)
    actions = torch.empty(n, H, dtype=torch.int32, device=device)
    for h, a in enumerate(cfg.heads):
        actions[:, h] = torch.randint(0, a, (n,), generator=g, device=device, dtype=torch.int32)
    xi = 0.15 * torch.randn(n, generator=g, device=device)
    logp_old = (-sum(math.log(a) for a in cfg.heads) - xi).float()
    return dict(rewards=r.float().contiguous(), values=values.contiguous(),
                dones=d.to(torch.uint8).contiguous(), obs=obs, actions=actions,
                logp_old=logp_old.contiguous(), n=n, Bk=Bk)
