"""Shared fixtures for the PPO-step parity tests: one seeded batch run through the CUDA path
(C ABI via the ctypes binding) and through the oracle, plus the C-T* comparison metrics."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth


KINK_MARGIN = 0.01


def kink_free_xi(cfg, xi, margin=KINK_MARGIN):
    """Move every log-ratio xi = log rho at least `margin` away from the clip kinks
    log(1 +- eps), where the PPO loss is not differentiable (DESIGN.md §3.4 reading R-K)."""
    xi = np.array(xi, dtype=np.float64)
    for k in (np.log(1 + cfg.clip_eps), np.log(1 - cfg.clip_eps)):
        close = np.abs(xi - k) < margin
        xi[close] = k + np.where(xi[close] >= k, margin, -margin)
    return xi


def make_inputs(cfg, seed=0, stress=False, head_gain=1.0, world=1, rank=0, margin=KINK_MARGIN):
    params = synth.make_params(cfg, seed, head_gain=head_gain)
    b = synth.make_batch(cfg, seed=seed, stress=stress, world=world, rank=rank)
    # parity recipe: behaviour log-prob = log pi_theta0(a) - xi, with xi
    # kept off the clip kinks so both sides take the same (exactly defined) branch
    xi = kink_free_xi(cfg, b["xi"], margin) if margin > 0 else b["xi"]
    b["logp_old"] = (oracle.log_pi(cfg, params, b["obs"], b["actions"]) - xi).astype(np.float32)
    return params, b


def to_dev(b):
    return {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda()
            for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}


def gpu_step(cfg, params, shards, apply=True, ctx=None, n_steps=1):
    """Run GAE -> adv_norm (global over all shards, virtual ranks) -> ppo_step on one GPU.
    With several shards and apply=False the per-shard gradients are summed in rank order."""
    import paper_2306_16688_b200 as P
    spec = P.NetSpec.from_config(cfg)
    devs = [to_dev(s) for s in shards]
    N = sum(s["n"] for s in shards)
    gae_out = []
    for d in devs:
        adv, ret, st = P.gae(d["rewards"], d["values"], d["dones"], cfg.gamma, cfg.lam)
        gae_out.append((adv.reshape(-1), ret.reshape(-1), st))
    allA = torch.cat([g[0] for g in gae_out])
    ms = P.adv_norm(allA) if len(shards) > 1 else P.adv_norm(gae_out[0][0], local_stats=gae_out[0][2])
    if ctx is None:
        ctx = P.PPOContext(spec, max_local_n=max(s["n"] for s in shards))
        ctx.load_params(torch.from_numpy(params).cuda())
    grads = None
    stats = None
    for _ in range(n_steps):
        for d, (adv, ret, _) in zip(devs, gae_out):
            stats = ctx.step(N, d["obs"], d["actions"], d["logp_old"], adv, ret, ms, apply=apply)
            if not apply:
                g = ctx.grads()
                grads = g if grads is None else grads + g
    torch.cuda.synchronize()
    out = dict(ctx=ctx, stats=P.decode_stats(stats), mean_std=ms.cpu().numpy(),
               adv=[g[0].cpu().numpy() for g in gae_out], ret=[g[1].cpu().numpy() for g in gae_out])
    out["bucket"] = (grads if grads is not None else ctx.grads()).cpu().numpy().astype(np.float64)
    out["params"] = ctx.params().cpu().numpy().astype(np.float64)
    m, v = ctx.adam_state()
    out["m"], out["v"] = m.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)
    return out


def tensor_slices(cfg):
    """(name, slice) of every W_l and b_l in the flat layout (C-A10)."""
    off, out = 0, []
    for l, (o, i) in enumerate(cfg.layer_shapes):
        nw = o * i
        out.append((f"W{l + 1}", slice(off, off + nw)))
        out.append((f"b{l + 1}", slice(off + nw, off + nw + o)))
        off += nw + o
    return out


def grad_errors(cfg, g, gref):
    """C-T3: per tensor relative L2 and max-abs-relative errors."""
    res = {}
    for name, sl in tensor_slices(cfg):
        a, r = g[sl], gref[sl]
        nr = np.linalg.norm(r)
        res[name] = (np.linalg.norm(a - r) / max(nr, 1e-30),
                     np.abs(a - r).max() / max(np.abs(r).max(), 1e-30))
    return res


def oracle_term_scales(cfg, params, shards, o):
    """Scale of each loss component for C-T4: mean |per-sample term| under the oracle."""
    lp = np.concatenate([oracle.log_pi(cfg, params, s["obs"], s["actions"]) for s in shards])
    lo = np.concatenate([s["logp_old"] for s in shards]).astype(np.float64)
    ahat = (np.concatenate(o["adv"]) - o["mean"]) / (o["std"] + 1e-8)
    rho = np.exp(lp - lo)
    N = o["N"]
    near = np.sum(np.minimum(np.abs(rho - (1 + cfg.clip_eps)), np.abs(rho - (1 - cfg.clip_eps))) <= 1e-3)
    return dict(pg=np.mean(np.abs(rho * ahat)), v=o["sums"][1] / N, ent=o["sums"][2] / N,
                kl=np.mean(np.abs(lp)), clip_near=near / N)


def near_kink(cfg, params, obs, actions, logp_old, margin=KINK_MARGIN / 2, v_old=None, ret=None,
              value_clip=0.0):
    """Samples whose loss is within `margin` of a non-differentiable point at `params`, by the
    oracle (DESIGN.md §3.3 R-K, §3.5 R-V): the log-ratio near log(1 +- eps), or (value clipping)
    |V - v_old| near the band edge or the two value losses within `margin` of a tie.
    The default margin is half the fixtures' (whose samples sit AT KINK_MARGIN, up to fp32
    rounding of logp_old) and still 5x the kernel's ~1e-3 log-prob error."""
    xi = oracle.log_pi(cfg, params, obs, actions) - np.asarray(logp_old, np.float64)
    near = np.zeros(xi.size, bool)
    for k in (np.log(1 + cfg.clip_eps), np.log(1 - cfg.clip_eps)):
        near |= np.abs(xi - k) < margin
    if value_clip > 0:
        V = oracle.forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, obs, separate=oracle.sep(cfg))[:, -1]
        vo = np.asarray(v_old, np.float64)
        R = np.asarray(ret, np.float64)
        d = V - vo
        vc = vo + np.clip(d, -value_clip, value_clip)
        near |= np.abs(np.abs(d) - value_clip) < margin
        near |= (np.abs(d) > value_clip) & (np.abs((vc - R) ** 2 - (V - R) ** 2) < margin)
    return near


def value_kink_free(cfg, params, b, value_clip, margin=KINK_MARGIN, rounds=20):
    """Nudge the rollout values (v_old = values rows 0..T-1, which also feed GAE) until no
    sample is within `margin` of a value-clip kink at `params` (fixture for R-V parity)."""
    b = dict(b)
    vals = np.array(b["values"], np.float32)
    T, Bk = vals.shape[0] - 1, vals.shape[1]
    V = oracle.forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"], separate=oracle.sep(cfg))[:, -1]
    for _ in range(rounds):
        _, r = oracle.gae(b["rewards"], vals, b["dones"], cfg.gamma, cfg.lam)
        vo = vals[:-1].reshape(-1).astype(np.float64)
        R = r.reshape(-1)
        d = V - vo
        vc = vo + np.clip(d, -value_clip, value_clip)
        bad = np.abs(np.abs(d) - value_clip) < margin
        bad |= (np.abs(d) > value_clip) & (np.abs((vc - R) ** 2 - (V - R) ** 2) < margin)
        if not bad.any():
            b["values"] = vals
            return b
        vals[:-1].reshape(-1)[bad] += np.float32(0.05)
    raise RuntimeError("value_kink_free: did not converge")
