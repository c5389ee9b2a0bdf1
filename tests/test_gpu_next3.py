"""NEXT-3 parity: value-loss clipping in the fused loss
epilogue, global gradient-norm clipping before Adam, and epochs x minibatches inside
srl_ppo_train_step -- each through the C ABI against the oracle."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import grad_errors, make_inputs, to_dev

pytestmark = pytest.mark.gpu

TOL = 2e-3
REDUCED = {"tiny": 4, "gfootball": 16, "hns": 4}


def _spec(cfg, **kw):
    import paper_2306_16688_b200 as P
    return dataclasses.replace(P.NetSpec.from_config(cfg), **kw)


def _ctx(cfg, params, n, **kw):
    import paper_2306_16688_b200 as P
    ctx = P.PPOContext(_spec(cfg, **kw), max_local_n=n)
    ctx.load_params(torch.from_numpy(np.ascontiguousarray(params, np.float32)).cuda())
    return ctx


def _check_grads(cfg, g, gref, tol=TOL):
    errs = grad_errors(cfg, g, gref)
    bad = {k: v for k, v in errs.items() if v[0] > tol or v[1] > tol}
    assert not bad, bad


def _value_clip_fixture(cfg, params, b, ev, seed):
    """v_old around the network's own V: |V - v_old| in [0, 0.15] (inside the band) or
    [0.25, 1] (outside), and for outside samples |l_c - l_v| >= 0.05, so the GPU (fp16 forward,
    |dV| ~ 1e-3) and the oracle take the same branch (the R-K kink argument)."""
    rng = np.random.default_rng(seed)
    n = b["n"]
    V = oracle.forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"])[:, -1]
    inside = rng.random(n) < 0.4
    mag = np.where(inside, rng.uniform(0.0, ev - 0.05, n), rng.uniform(ev + 0.05, 1.0, n))
    vold = (V - np.where(rng.random(n) < 0.5, -mag, mag)).astype(np.float32).astype(np.float64)
    a, r = oracle.gae(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam)
    ahat, _, _ = oracle.adv_norm(a.reshape(-1))
    ret = r.reshape(-1).copy()
    for i in np.nonzero(~inside)[0]:
        d = V[i] - vold[i]
        vc = vold[i] + np.clip(d, -ev, ev)
        while abs((vc - ret[i]) ** 2 - (V[i] - ret[i]) ** 2) < 0.05:
            ret[i] += 0.1
    f32 = lambda x: np.asarray(x, np.float32)
    return f32(ahat), f32(ret), f32(vold), (V - vold, ret)


@pytest.mark.parametrize("name", list(REDUCED))
def test_value_clip_grad_parity(name):
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=31)
    ev = 0.2
    ahat, ret, vold, (d, r64) = _value_clip_fixture(cfg, params, b, ev, 31)
    n = b["n"]
    ctx = _ctx(cfg, params, n, value_clip=ev)
    dv = to_dev(b)
    t = lambda x: torch.from_numpy(x).cuda()
    import paper_2306_16688_b200 as P
    st = P.decode_stats(ctx.step(n, dv["obs"], dv["actions"], dv["logp_old"], t(ahat), t(ret),
                                 None, apply=False, v_old=t(vold)))
    G = ctx.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
    g, sums, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"],
                                      b["actions"], b["logp_old"], ahat, ret, cfg.clip_eps,
                                      cfg.value_coef, cfg.entropy_coef, grad_scale=1.0 / n,
                                      v_old=vold, value_clip=ev)
    _check_grads(cfg, G, g)
    assert abs(st["value_loss"] - sums[1] / n) <= TOL * sums[1] / n
    # the clip changed something: the plain loss differs
    g0, s0, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"],
                                     b["actions"], b["logp_old"], ahat, ret, cfg.clip_eps,
                                     cfg.value_coef, cfg.entropy_coef, grad_scale=1.0 / n)
    assert s0[1] < sums[1] and np.linalg.norm(g0 - g) > 10 * TOL * np.linalg.norm(g)


def test_value_clip_needs_v_old():
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("tiny")
    params, b = make_inputs(cfg, seed=1)
    ctx = _ctx(cfg, params, b["n"], value_clip=0.2)
    dv = to_dev(b)
    z = torch.zeros(b["n"], device="cuda")
    with pytest.raises(P.SrlError):
        ctx.step(b["n"], dv["obs"], dv["actions"], dv["logp_old"], z, z, None, apply=False)


@pytest.mark.parametrize("frac", [0.3, 2.0])
def test_grad_norm_clip_identical_g(frac):
    """The kernel's pre-clip norm matches ||G||; Adam on the kernel's own G after the oracle's
    clip (identical-G, as test_ppo_step_apply_adam) matches the kernel's update.  frac = 2:
    max_norm above the norm, nothing is scaled."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("gfootball").with_(B=16)
    params, b = make_inputs(cfg, seed=9)
    dv = to_dev(b)
    n = b["n"]
    probe = _ctx(cfg, params, n)
    probe.train_step(n, dv["rewards"], dv["values"], dv["dones"], dv["obs"], dv["actions"],
                     dv["logp_old"])
    n0 = float(np.linalg.norm(probe.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]))
    ctx = _ctx(cfg, params, n, max_grad_norm=frac * n0)
    st = P.decode_stats(ctx.train_step(n, dv["rewards"], dv["values"], dv["dones"], dv["obs"],
                                       dv["actions"], dv["logp_old"]))
    G = ctx.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
    assert abs(st["grad_norm"] - np.linalg.norm(G)) <= 1e-6 * np.linalg.norm(G)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    assert abs(st["grad_norm"] - np.linalg.norm(o["grad"])) <= TOL * np.linalg.norm(o["grad"])
    Gc = G.copy()
    oracle.clip_grad_norm(Gc, frac * n0)
    p = params.astype(np.float64).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam(p, m, v, Gc, 1, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    got = ctx.params().cpu().numpy().astype(np.float64)
    assert np.linalg.norm((got - params) - (p - params)) <= 1e-5 * np.linalg.norm(p - params)
    mg = ctx.adam_state()[0].cpu().numpy().astype(np.float64)
    assert np.abs(mg - m).max() <= 1e-6 * np.abs(m).max()
    assert st["step"] == 1


@pytest.mark.parametrize("E,M", [(2, 1), (1, 3), (2, 2)])
def test_epochs_minibatches_equal_composed_steps(E, M):
    """srl_ppo_train_step with E x M updates is bit-identical to E x M srl_ppo_step calls on
    the minibatch row ranges (R-M), and each update's gradient matches the oracle's gradient
    of that minibatch at the parameters the update started from.  Value clipping and
    gradient-norm clipping on, so all of NEXT-3 runs in one step."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("gfootball").with_(B=20)
    params, b = make_inputs(cfg, seed=13)
    n = b["n"]
    kw = dict(epochs=E, minibatches=M, value_clip=0.2, max_grad_norm=0.05)
    dv = to_dev(b)
    a = _ctx(cfg, params, n, **kw)
    st = P.decode_stats(a.train_step(n, dv["rewards"], dv["values"], dv["dones"], dv["obs"],
                                     dv["actions"], dv["logp_old"]))
    c = _ctx(cfg, params, n, **kw)
    adv, ret, gst = P.gae(dv["rewards"], dv["values"], dv["dones"], cfg.gamma, cfg.lam)
    adv, ret = adv.reshape(-1), ret.reshape(-1)
    ms = P.adv_norm(adv, local_stats=gst)
    vold = dv["values"][:-1].reshape(-1)
    mu, sd = ms.cpu().numpy()
    for e in range(E):
        for lo, hi in oracle.minibatch_bounds(n, M):
            p0 = c.params().cpu().numpy().astype(np.float64)
            c.step(hi - lo, dv["obs"][lo:hi], dv["actions"][lo:hi], dv["logp_old"][lo:hi],
                   adv[lo:hi], ret[lo:hi], ms, apply=True, v_old=vold[lo:hi])
            G = c.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
            ah = (adv[lo:hi].cpu().numpy().astype(np.float64) - mu) / (sd + 1e-8)
            g, _, _ = oracle.loss_and_grad(
                cfg.obs_dim, cfg.hidden, cfg.heads, p0, b["obs"][lo:hi], b["actions"][lo:hi],
                b["logp_old"][lo:hi], ah, ret[lo:hi].cpu().numpy(), cfg.clip_eps,
                cfg.value_coef, cfg.entropy_coef, v_old=vold[lo:hi].cpu().numpy(),
                value_clip=0.2)
            # kink flips of the value clip are possible at later updates (params moved):
            # compare at the C-T3 bound on the whole vector
            assert np.linalg.norm(G - g) <= 5 * TOL * np.linalg.norm(g)
    torch.cuda.synchronize()
    assert torch.equal(a.params(), c.params()) and torch.equal(a.grads(), c.grads())
    assert st["step"] == E * M
    assert st["n_global"] == oracle.minibatch_bounds(n, M)[-1][1] - oracle.minibatch_bounds(n, M)[-1][0]
    assert st["grad_norm"] > 0.05                  # clipping was active


def test_minibatches_reject_bad_sizes():
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("tiny").with_(B=2)
    params, b = make_inputs(cfg, seed=4)
    dv = to_dev(b)
    ctx = _ctx(cfg, params, b["n"], minibatches=b["n"] + 1)
    with pytest.raises(P.SrlError):
        ctx.train_step(b["n"], dv["rewards"], dv["values"], dv["dones"], dv["obs"],
                       dv["actions"], dv["logp_old"])
    ctx2 = _ctx(cfg, params, b["n"], minibatches=2)
    with pytest.raises(P.SrlError):              # unequal shards would need N_k per rank
        ctx2.train_step(2 * b["n"], dv["rewards"], dv["values"], dv["dones"], dv["obs"],
                        dv["actions"], dv["logp_old"])
