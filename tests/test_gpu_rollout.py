"""NEXT-2 parity: srl_policy_rollout (forward + sampling epilogue) through the C ABI against the
oracle's rollout (reading R-S).

The action is an integer decided by floating point: the kernel decides in fp32 from fp16-GEMM
logits, the oracle in double.  Where the oracle's decision margin (distance of u from a CDF
boundary, or the gap between the two largest logits) exceeds the logits' error bound the
actions must be identical; inside it the kernel's action must be one the margin allows (an
adjacent CDF bucket, or a near-maximal logit).  logp / value within the C-T tolerances."""
import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import make_inputs

pytestmark = pytest.mark.gpu

MARGIN = 5e-3


def _ctx(cfg, params, n):
    import paper_2306_16688_b200 as P
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=n)
    ctx.load_params(torch.from_numpy(np.ascontiguousarray(params, np.float32)).cuda())
    return ctx


def _check(cfg, params, obs, got, ref, deterministic):
    act, lp, val = (x.cpu().numpy() for x in got)
    ract, rlp, rval, mg = ref
    safe = mg > MARGIN
    assert np.array_equal(act[safe], ract[safe]), np.argwhere(act != ract)[:5]
    if deterministic:                                    # unsafe: a near-maximal logit
        z = oracle.forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, obs)
        s = 0
        for h, a in enumerate(cfg.heads):
            zz = z[:, s:s + a]
            pick = zz[np.arange(len(zz)), act[:, h]]
            assert np.all(pick >= zz.max(1) - MARGIN)
            s += a
    else:
        assert np.all(np.abs(act.astype(np.int64) - ract) <= 1)
    same = np.all(act == ract, axis=1)
    assert same.mean() > 0.98
    # logp of the kernel's own action under the oracle's double forward
    cls = type("c", (), dict(obs_dim=cfg.obs_dim, hidden=cfg.hidden, heads=cfg.heads))
    lp_ref = oracle.log_pi(cls(), params, obs, act)
    assert np.max(np.abs(lp - lp_ref)) <= 2e-3 * (1 + np.abs(lp_ref).mean())
    assert np.max(np.abs(val - rval)) <= 2e-3 * (1 + np.abs(rval).mean())


@pytest.mark.parametrize("name", ["tiny", "atari", "gfootball", "hns"])
@pytest.mark.parametrize("deterministic", [False, True])
def test_rollout_parity(name, deterministic):
    cfg = synth.get_config(name)
    cfg = cfg.with_(B=min(cfg.B, 12 * cfg.agents))
    params, b = make_inputs(cfg, seed=23, head_gain=3.0)
    n = b["n"]
    ctx = _ctx(cfg, params, n)
    obs = torch.from_numpy(b["obs"]).cuda()
    keys = torch.from_numpy((np.arange(n, dtype=np.int64) * 2654435761) % (1 << 40)).cuda()
    got = ctx.rollout(obs, keys=keys, seed=99, deterministic=deterministic)
    torch.cuda.synchronize()
    ref = oracle.rollout(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"], seed=99,
                         keys=keys.cpu().numpy().astype(np.uint64), deterministic=deterministic)
    _check(cfg, params, b["obs"], got, ref, deterministic)


def test_rollout_row_independent_and_key_default():
    """A request's result depends only on (obs row, key): permuting rows together with their
    keys permutes the outputs bit for bit; keys = NULL means key = row index."""
    cfg = synth.get_config("gfootball").with_(B=16)
    params, b = make_inputs(cfg, seed=2)
    n = b["n"]
    ctx = _ctx(cfg, params, n)
    obs = torch.from_numpy(b["obs"]).cuda()
    keys = torch.arange(n, dtype=torch.int64, device="cuda")
    a1, l1, v1 = ctx.rollout(obs, keys=keys, seed=5)
    a0, l0, v0 = ctx.rollout(obs, seed=5)
    assert torch.equal(a0, a1) and torch.equal(l0, l1) and torch.equal(v0, v1)
    perm = torch.from_numpy(np.random.default_rng(0).permutation(n)).cuda()
    a2, l2, v2 = ctx.rollout(obs[perm].contiguous(), keys=keys[perm].contiguous(), seed=5)
    assert torch.equal(a2, a1[perm]) and torch.equal(l2, l1[perm]) and torch.equal(v2, v1[perm])


def test_rollout_fullsize_sampled():
    """Atari-shaped full batch (n = 131072) in one call; 3000 sampled rows against the oracle."""
    cfg = synth.get_config("atari")
    params = synth.make_params(cfg, 0)
    b = synth.make_batch(cfg, seed=4, with_obs=True)
    n = b["n"]
    ctx = _ctx(cfg, params, n)
    obs = torch.from_numpy(b["obs"]).cuda()
    act, lp, val = ctx.rollout(obs, seed=1234)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(1).choice(n, 3000, replace=False))
    ref = oracle.rollout(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"][rows], seed=1234,
                         keys=rows.astype(np.uint64))
    ri = torch.from_numpy(rows).cuda()
    _check(cfg, params, b["obs"][rows], (act[ri], lp[ri], val[ri]), ref, False)
