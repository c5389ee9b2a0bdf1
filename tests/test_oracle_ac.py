"""Pins for the NEXT-3 separate actor / critic trunks in the oracle (oracle_*_ac; SURVEY.md
§8(f) NEXT-3; DESIGN.md §3.5 reading R-AC).

Against: central finite differences of the per-sample losses (rel <= 1e-6);
the shared-trunk oracle (with tied trunks the two-trunk net IS the shared net whose head is
[W_pi; w_v], so outputs agree exactly and the shared trunk's gradient is the SUM of the two
trunks' gradients -- a transposed block, a swapped trunk or a dropped path fails it); and the
structural zeros (c_v = 0: no critic gradient; A_hat = 0 and c_e = 0: no actor gradient).
"""
import math

import numpy as np
import pytest

import oracle
import synth

NETS = [(4, (8, 8), (2,)), (5, (6, 7), (3, 2)), (3, (5,), (4, 2, 2))]


def _params(net, seed, separate, scale=1.5):
    P = oracle.param_count(*net, separate=separate)
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, P) * scale / math.sqrt(net[0])


def _batch(net, n, seed):
    obs_dim, hidden, heads = net
    rng = np.random.default_rng(seed)
    obs = rng.normal(size=(n, obs_dim))
    act = np.stack([rng.integers(0, a, n) for a in heads], 1).astype(np.int32)
    return obs, act, rng


def _split(net, p):
    """(actor trunk, W_pi + b_pi, critic trunk, w_v + b_v) slices of the R-AC layout."""
    obs_dim, hidden, heads = net
    d = (obs_dim,) + tuple(hidden)
    T = sum(d[i + 1] * d[i] + d[i + 1] for i in range(len(hidden)))
    A, h = sum(heads), d[-1]
    o_pi = T
    o_c = T + A * h + A
    o_v = o_c + T
    return p[:T], p[o_pi:o_c], p[o_c:o_v], p[o_v:]


def test_param_count_closed_form():
    for net in NETS:
        obs_dim, hidden, heads = net
        d = (obs_dim,) + hidden
        T = sum(d[i + 1] * d[i] + d[i + 1] for i in range(len(hidden)))
        A = sum(heads)
        assert oracle.param_count(*net, separate=True) == 2 * T + A * d[-1] + A + d[-1] + 1
    for name in ("atari", "hns"):
        cfg = synth.get_config(name).with_(separate_critic=True)
        assert cfg.n_params == oracle.param_count(cfg.obs_dim, cfg.hidden, cfg.heads, separate=True)


@pytest.mark.parametrize("net", NETS)
def test_tied_trunks_equal_shared_net(net):
    obs_dim, hidden, heads = net
    A = sum(heads)
    h = hidden[-1]
    ps = _params(net, 3, False)                    # shared: trunk, head [A+1][h] + [A+1]
    d = (obs_dim,) + hidden
    T = sum(d[i + 1] * d[i] + d[i + 1] for i in range(len(hidden)))
    trunk, head = ps[:T], ps[T:]
    Wh, bh = head[:(A + 1) * h].reshape(A + 1, h), head[(A + 1) * h:]
    pac = np.concatenate([trunk, Wh[:A].ravel(), bh[:A], trunk, Wh[A:].ravel(), bh[A:]])
    n = 9
    obs, act, rng = _batch(net, n, 4)
    zs = oracle.forward(*net, ps, obs)
    za = oracle.forward(*net, pac, obs, separate=True)
    assert np.array_equal(zs, za)
    lo = rng.normal(size=n) - 1.0
    ah, ret = rng.normal(size=n), rng.normal(size=n)
    gs, ss, _ = oracle.loss_and_grad(*net, ps, obs, act, lo, ah, ret)
    ga, sa, _ = oracle.loss_and_grad(*net, pac, obs, act, lo, ah, ret, separate=True)
    assert np.array_equal(ss, sa)
    at, apih, ct, vh = _split(net, ga)
    tol = 1e-12 * np.abs(gs).max()
    assert np.abs((at + ct) - gs[:T]).max() <= tol          # shared trunk = actor + critic
    gWh = gs[T:T + (A + 1) * h].reshape(A + 1, h)
    gbh = gs[T + (A + 1) * h:]
    assert np.abs(apih - np.concatenate([gWh[:A].ravel(), gbh[:A]])).max() <= tol
    assert np.abs(vh - np.concatenate([gWh[A:].ravel(), gbh[A:]])).max() <= tol


@pytest.mark.parametrize("net", NETS)
def test_structural_zeros(net):
    p = _params(net, 5, True)
    n = 7
    obs, act, rng = _batch(net, n, 6)
    lo = rng.normal(size=n) - 1.0
    ret = rng.normal(size=n)
    g, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, rng.normal(size=n), ret, 0.2, 0.0, 0.01,
                                   separate=True)
    at, apih, ct, vh = _split(net, g)
    assert not ct.any() and not vh.any()                     # c_v = 0: the critic gets nothing
    assert np.abs(at).max() > 0 and np.abs(apih).max() > 0
    g, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, np.zeros(n), ret, 0.2, 0.5, 0.0,
                                   separate=True)
    at, apih, ct, vh = _split(net, g)
    assert not at.any() and not apih.any()                   # no policy / entropy term
    assert np.abs(ct).max() > 0 and np.abs(vh).max() > 0


@pytest.mark.parametrize("net,clip,vclip", [(NETS[0], 10.0, 0.0), (NETS[1], 0.2, 0.0),
                                            (NETS[2], 0.2, 0.3)])
def test_finite_difference_gradient(net, clip, vclip):
    """Central FD, step 1e-5, relative error <= 1e-6, kink-free fixture (policy ratio and,
    with value clipping, |V - v_old| kept away from the band edge and the branch tie)."""
    obs_dim, hidden, heads = net
    p = _params(net, 8, True)
    n = 10
    obs, act, rng = _batch(net, n, 9)
    cls = type("c", (), dict(obs_dim=obs_dim, hidden=hidden, heads=heads, separate_critic=True))
    lp = oracle.log_pi(cls(), p, obs, act)
    rho = np.exp(rng.uniform(-0.5, 0.5, n))
    for k in (1 + clip, 1 - clip):
        close = np.abs(rho - k) < 5e-3
        rho[close] = k + 0.02
    lo = lp - np.log(rho)
    ah, ret = rng.normal(size=n), rng.normal(size=n)
    V = oracle.forward(*net, p, obs, separate=True)[:, -1]
    vold = V - np.where(rng.random(n) < 0.5, 0.1, 0.6) * np.sign(rng.normal(size=n))
    if vclip > 0:                                            # move ties / edges away
        for i in range(n):
            d = V[i] - vold[i]
            vc = vold[i] + np.clip(d, -vclip, vclip)
            while abs(d) > vclip and abs((vc - ret[i]) ** 2 - (V[i] - ret[i]) ** 2) < 1e-2:
                ret[i] += 0.1
    kw = dict(v_old=vold if vclip > 0 else None, value_clip=vclip, separate=True)

    def total(pp):
        _, _, ps = oracle.loss_and_grad(*net, pp, obs, act, lo, ah, ret, clip, 0.5, 0.01,
                                        want_per_sample=True, **kw)
        return ps.sum() / n

    g, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, ah, ret, clip, 0.5, 0.01, **kw)
    h = 1e-5
    fd = np.empty_like(p)
    for k in range(p.size):
        pp, pm = p.copy(), p.copy()
        pp[k] += h
        pm[k] -= h
        fd[k] = (total(pp) - total(pm)) / (2 * h)
    err = np.abs(g - fd)
    tol = 1e-6 * np.maximum(np.abs(fd), np.abs(fd).max() * 1e-3)
    assert np.all(err <= tol), float((err / np.maximum(np.abs(fd), 1e-12)).max())


def test_ppo_step_dispatches_on_config():
    """oracle.ppo_step on a separate_critic config uses the two-trunk network end to end."""
    from ppo_harness import make_inputs
    cfg = synth.get_config("tiny").with_(separate_critic=True)
    params, b = make_inputs(cfg, seed=1)
    assert params.size == cfg.n_params
    o = oracle.ppo_step(cfg, params, [b], apply=True)
    assert o["grad"].size == cfg.n_params and np.all(np.isfinite(o["params"]))
    net = (cfg.obs_dim, cfg.hidden, cfg.heads)
    ahat = (o["adv"][0] - o["mean"]) / (o["std"] + 1e-8)
    g, _, _ = oracle.loss_and_grad(*net, params, b["obs"], b["actions"], b["logp_old"], ahat,
                                   o["ret"][0], cfg.clip_eps, cfg.value_coef, cfg.entropy_coef,
                                   grad_scale=1.0 / o["N"], separate=True)
    assert np.array_equal(g, o["grad"])
