"""Parity at BASELINE.json's full Atari-shaped size (T=128, B=1024, n=131072), in the launch
configuration bench.py times.  The oracle runs over 16 column shards in parallel host processes
and its per-shard gradients are summed in rank order (C-5, pinned by
tests/test_oracle_adam_kshard.py), so the whole batch is compared element by element.

* kink-free recipe (DESIGN.md §3.3 R-K): gradients per tensor within 2e-3, loss terms within
  2e-3 of their scale;
* the bench recipe (uniform behaviour policy, wide rho): clip decisions may differ only for
  samples whose oracle log-ratio lies within 0.01 of a kink.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CFG = synth.get_config("atari")
W = 16
PARAMS = synth.make_params(CFG, 0)


def _lp_shard(r):
    b = synth.make_batch(CFG, seed=0, world=W, rank=r)
    return r, oracle.log_pi(CFG, PARAMS, b["obs"], b["actions"])


def _grad_shard(args):
    r, lo, mean, std = args
    b = synth.make_batch(CFG, seed=0, world=W, rank=r)
    adv, ret = oracle.gae(b["rewards"], b["values"], b["dones"], CFG.gamma, CFG.lam)
    g, sums, _ = oracle.loss_and_grad(CFG.obs_dim, CFG.hidden, CFG.heads, PARAMS, b["obs"],
                                      b["actions"], lo, (adv.reshape(-1) - mean) / (std + 1e-8),
                                      ret.reshape(-1), CFG.clip_eps, CFG.value_coef,
                                      CFG.entropy_coef, grad_scale=1.0 / CFG.N)
    return r, g, sums


def _to_full(parts):
    Bk = CFG.B // W
    return np.concatenate([p.reshape(CFG.T, Bk) for p in parts], axis=1).reshape(-1)


def _to_shards(x):
    Bk = CFG.B // W
    x = x.reshape(CFG.T, CFG.B)
    return [np.ascontiguousarray(x[:, r * Bk:(r + 1) * Bk]).reshape(-1) for r in range(W)]


@pytest.fixture(scope="module")
def setup():
    full = synth.make_batch(CFG, seed=0)
    ra, _ = oracle.gae(full["rewards"], full["values"], full["dones"], CFG.gamma, CFG.lam)
    _, mean, std = oracle.adv_norm(ra)
    pool = mp.get_context("fork").Pool(min(W, os.cpu_count() or 1))
    lp = _to_full([x[1] for x in sorted(pool.map(_lp_shard, range(W)), key=lambda x: x[0])])
    yield full, mean, std, lp, pool
    pool.close()


def _gpu(full, logp_old):
    import paper_2306_16688_b200 as P
    d = {k: torch.from_numpy(np.ascontiguousarray(full[k])).cuda()
         for k in ("rewards", "values", "dones", "obs", "actions")}
    d["logp_old"] = torch.from_numpy(logp_old).cuda()
    adv, ret, st = P.gae(d["rewards"], d["values"], d["dones"], CFG.gamma, CFG.lam)
    ms = P.adv_norm(adv.view(-1), local_stats=st)
    ctx = P.PPOContext(P.NetSpec.from_config(CFG), max_local_n=full["n"])
    ctx.load_params(torch.from_numpy(PARAMS).cuda())
    stats = P.decode_stats(ctx.step(full["n"], d["obs"], d["actions"], d["logp_old"], adv.view(-1),
                                    ret.view(-1), ms, apply=False))
    return ms.cpu().numpy(), stats, ctx.grads().cpu().numpy().astype(np.float64)


def test_atari_full_batch_gradient_kink_free(setup):
    from ppo_harness import grad_errors, kink_free_xi
    full, mean, std, lp, pool = setup
    xi = lp - synth.logp_old_uniform_policy(CFG, full["xi"]).astype(np.float64)
    lo32 = (lp - kink_free_xi(CFG, xi)).astype(np.float32)
    ms, stats, G = _gpu(full, lo32)
    assert abs(ms[0] - mean) <= 1e-6 * std and abs(ms[1] - std) <= 1e-6 * std
    jobs = [(r, s.astype(np.float64), mean, std) for r, s in enumerate(_to_shards(lo32))]
    res = sorted(pool.map(_grad_shard, jobs), key=lambda x: x[0])
    gref = np.zeros(CFG.n_params)
    sums = np.zeros(5)
    for _, g, s in res:                      # rank order
        gref += g
        sums += s
    errs = grad_errors(CFG, G[:CFG.n_params], gref)
    assert all(v[0] <= 2e-3 and v[1] <= 2e-3 for v in errs.values()), errs
    ref = sums / CFG.N
    rho = np.exp(lp - lo32.astype(np.float64))
    ahat = (oracle.gae(full["rewards"], full["values"], full["dones"], CFG.gamma, CFG.lam)[0].reshape(-1)
            - mean) / (std + 1e-8)
    assert abs(stats["policy_loss"] - ref[0]) <= 2e-3 * np.mean(np.abs(rho * ahat))
    assert abs(stats["value_loss"] - ref[1]) <= 2e-3 * ref[1]
    assert abs(stats["entropy"] - ref[2]) <= 2e-3 * ref[2]
    assert abs(stats["clip_fraction"] - ref[3]) <= 1.0 / CFG.N
    assert stats["nonfinite"] == 0 and stats["n_global"] == CFG.N


def test_atari_full_batch_bench_recipe_clip_decisions(setup):
    full, mean, std, lp, pool = setup
    lo32 = synth.logp_old_uniform_policy(CFG, full["xi"]).astype(np.float32)
    _, stats, _ = _gpu(full, lo32)
    xi = lp - lo32.astype(np.float64)
    ref = np.mean(np.abs(np.exp(xi) - 1.0) > CFG.clip_eps)
    near = sum(np.sum(np.abs(xi - np.log(1 + s * CFG.clip_eps)) < 0.01) for s in (1, -1))
    assert abs(stats["clip_fraction"] - ref) <= near / CFG.N + 1e-7
