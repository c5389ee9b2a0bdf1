"""Pins for oracle C-3 (forward) and C-4 (PPO loss and gradient).

Against: SPEC.md's stated properties, the
hand-derived single-transition values in tests/golden/ppo_single_transition.json, and
central finite differences of the per-sample losses (the gradient is pinned by the loss,
so a dropped term, sign or transposed index in the backprop fails FD).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _net_params(obs_dim, hidden, heads, seed, scale=1.0):
    P = oracle.param_count(obs_dim, hidden, heads)
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, P) * scale / math.sqrt(max(obs_dim, 1))


def _batch(n, obs_dim, heads, seed):
    rng = np.random.default_rng(seed)
    obs = rng.normal(size=(n, obs_dim))
    act = np.stack([rng.integers(0, a, n) for a in heads], 1).astype(np.int32)
    return obs, act, rng


def _total_loss(net, params, obs, act, lo, ah, ret, clip, cv, ce):
    _, _, ps = oracle.loss_and_grad(*net, params, obs, act, lo, ah, ret, clip, cv, ce,
                                    want_per_sample=True)
    return ps.sum() / ps.size


def test_golden_single_transition():
    g = json.load(open(os.path.join(GOLD, "ppo_single_transition.json")))
    env = {"log": math.log}
    env["H"] = eval(g["H"], {}, env)
    net = (g["net"]["obs_dim"], tuple(g["net"]["hidden"]), tuple(g["net"]["heads"]))
    params = np.array(eval(g["params"], {}, env))
    obs = np.array(g["obs"], float)
    for c in g["cases"]:
        lo = np.array([eval(c["logp_old"], {}, env)])
        grad, sums, ps = oracle.loss_and_grad(
            *net, params, obs, np.array([[c["action"]]], np.int32), lo,
            np.array([c["adv_hat"]]), np.array([c["ret"]]), **g["coef"], grad_scale=1.0,
            want_per_sample=True)
        assert abs(ps[0] - eval(c["loss"], {}, env)) < 1e-14, c["name"]
        exp_sums = [eval(s, {}, env) for s in c["sums"]]
        np.testing.assert_allclose(sums, exp_sums, rtol=0, atol=1e-14)
        dz = np.array([eval(s, {}, env) for s in c["dz"]])
        # layout: W[3][1] (x = 1, so dW = dz) then b[3] (db = dz)
        np.testing.assert_allclose(grad, np.concatenate([dz, dz]), rtol=0, atol=1e-14)


def test_zero_net_uniform_logits_and_entropy():
    heads = (11, 11, 11, 2, 2)
    net = (6, (8, 8), heads)
    P = oracle.param_count(*net)
    obs, act, _ = _batch(5, 6, heads, 0)
    z = oracle.forward(*net, np.zeros(P), obs)
    assert np.array_equal(z, np.zeros_like(z))
    _, sums, _ = oracle.loss_and_grad(*net, np.zeros(P), obs, act, np.zeros(5), np.zeros(5),
                                      np.zeros(5))
    assert abs(sums[2] / 5 - sum(math.log(a) for a in heads)) < 1e-13   # S:L622 ln n per head


def test_batch_row_equals_single_call():
    net = (5, (16, 12), (4,))
    p = _net_params(*net, 1)
    obs, _, _ = _batch(9, 5, (4,), 1)
    z = oracle.forward(*net, p, obs)
    for i in range(9):
        assert np.array_equal(z[i], oracle.forward(*net, p, obs[i:i + 1])[0])


def test_no_hidden_layer_is_affine_map():
    """L=0 reduces to z = W x + b, checked with numpy's matmul (library routine)."""
    net = (7, (), (3, 2))
    p = _net_params(*net, 2)
    obs, _, _ = _batch(11, 7, (3, 2), 2)
    W = p[:6 * 7].reshape(6, 7)
    b = p[6 * 7:]
    np.testing.assert_allclose(oracle.forward(*net, p, obs), obs @ W.T + b, rtol=0, atol=1e-14)


def test_identity_ratio_policy_term_is_minus_mean_adv():
    """new params == old params -> rho = 1, clip_fraction 0, pg term = -mean(A)."""
    from synth import get_config
    cfg = get_config("tiny")
    p = _net_params(cfg.obs_dim, cfg.hidden, cfg.heads, 3)
    obs, act, rng = _batch(32, cfg.obs_dim, cfg.heads, 3)
    lo = oracle.log_pi(cfg, p, obs, act)
    ah = rng.normal(size=32)
    _, sums, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, p, obs, act, lo, ah,
                                      rng.normal(size=32))
    assert sums[3] == 0.0
    assert abs(sums[0] / 32 + ah.mean()) < 1e-14
    assert abs(sums[4]) < 1e-13


def test_zero_advantage_no_policy_gradient():
    """A = 0 -> only value and entropy terms move: the gradient equals the one
    with clip_eps changed arbitrarily and with logp_old changed arbitrarily."""
    net = (4, (8,), (3,))
    p = _net_params(*net, 4)
    obs, act, rng = _batch(10, 4, (3,), 4)
    ret = rng.normal(size=10)
    g1, _, _ = oracle.loss_and_grad(*net, p, obs, act, rng.normal(size=10), np.zeros(10), ret)
    g2, _, _ = oracle.loss_and_grad(*net, p, obs, act, rng.normal(size=10) * 5, np.zeros(10),
                                    ret, clip_eps=0.01)
    np.testing.assert_allclose(g1, g2, rtol=0, atol=1e-15)


def test_far_clipped_positive_adv_zero_policy_gradient():
    """rho >> 1+eps with A > 0: the clipped branch is constant, so the policy gradient is 0:
    the gradient equals the one at A = 0 (value/entropy terms only)."""
    net = (4, (8,), (3,))
    p = _net_params(*net, 5)
    obs, act, rng = _batch(6, 4, (3,), 5)
    ret = rng.normal(size=6)
    lo = oracle.log_pi(type("c", (), dict(obs_dim=4, hidden=(8,), heads=(3,)))(), p, obs, act) - 3.0
    g1, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, np.full(6, 2.0), ret)
    g0, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, np.zeros(6), ret)
    np.testing.assert_allclose(g1, g0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("net,clip", [
    ((4, (8, 8), (2,)), 10.0),            # clipping effectively off
    ((5, (6, 7), (3, 2)), 10.0),          # multi-head
    ((4, (8, 8), (2,)), 0.2),             # clipping on, kink-free fixture
    ((3, (5,), (4, 2, 2)), 0.2),
    ((6, (), (3,)), 0.2),                 # no hidden layer
])
def test_finite_difference_gradient(net, clip):
    """Central FD, step 1e-5, relative error <= 1e-6."""
    obs_dim, hidden, heads = net
    p = _net_params(*net, 6, scale=1.5)
    n = 12
    obs, act, rng = _batch(n, obs_dim, heads, 6)
    cls = type("c", (), dict(obs_dim=obs_dim, hidden=hidden, heads=heads))
    lp = oracle.log_pi(cls(), p, obs, act)
    # ratios spread around 1 but at least 1e-3 away from the clip kinks 1 +- clip
    rho = np.exp(rng.uniform(-0.5, 0.5, n))
    for k in (1 + clip, 1 - clip):
        close = np.abs(rho - k) < 5e-3
        rho[close] = k + 0.02
    lo = lp - np.log(rho)
    ah = rng.normal(size=n)
    ret = rng.normal(size=n)
    cv, ce = 0.5, 0.01
    grad, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, ah, ret, clip, cv, ce)
    h = 1e-5
    fd = np.empty_like(p)
    for k in range(p.size):
        pp, pm = p.copy(), p.copy()
        pp[k] += h
        pm[k] -= h
        fd[k] = (_total_loss(net, pp, obs, act, lo, ah, ret, clip, cv, ce)
                 - _total_loss(net, pm, obs, act, lo, ah, ret, clip, cv, ce)) / (2 * h)
    err = np.abs(grad - fd)
    tol = 1e-6 * np.maximum(np.abs(fd), np.abs(fd).max() * 1e-3)
    assert np.all(err <= tol), float((err / np.maximum(np.abs(fd), 1e-12)).max())


def test_single_head_equals_multi_head_with_one_head():
    net = (4, (8,), (5,))
    p = _net_params(*net, 7)
    obs, act, rng = _batch(8, 4, (5,), 7)
    args = (rng.normal(size=8), rng.normal(size=8), rng.normal(size=8))
    g1, s1, _ = oracle.loss_and_grad(*net, p, obs, act, *args)
    g2, s2, _ = oracle.loss_and_grad(4, [8], [5], p, obs, act.reshape(8, 1), *args)
    assert np.array_equal(g1, g2) and np.array_equal(s1, s2)


def test_gradient_additive_over_samples():
    """Gradient of the sum of two losses == sum of the gradients (S:L590 linearity)."""
    net = (4, (8, 6), (3,))
    p = _net_params(*net, 8)
    obs, act, rng = _batch(10, 4, (3,), 8)
    lo, ah, rt = rng.normal(size=10) - 1, rng.normal(size=10), rng.normal(size=10)
    g, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, ah, rt, grad_scale=1.0)
    ga, _, _ = oracle.loss_and_grad(*net, p, obs[:4], act[:4], lo[:4], ah[:4], rt[:4], grad_scale=1.0)
    gb, _, _ = oracle.loss_and_grad(*net, p, obs[4:], act[4:], lo[4:], ah[4:], rt[4:], grad_scale=1.0)
    np.testing.assert_allclose(g, ga + gb, rtol=1e-13, atol=1e-15)
