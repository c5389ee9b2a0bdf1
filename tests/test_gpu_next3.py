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


def _probe_grad(cfg, p0, n_mb, obs, actions, logp_old, adv, ret, ms, vold, keep, **kw):
    """The kernel's gradient at parameters p0 over the kept rows of one minibatch (padding
    mask = the rows away from every kink), mean over the minibatch's n_mb rows."""
    probe = _ctx(cfg, p0.astype(np.float32), n_mb, **kw)
    vm = torch.from_numpy(keep.astype(np.uint8)).cuda()
    probe.step(n_mb, obs, actions, logp_old, adv, ret, ms, apply=False, v_old=vold, valid=vm)
    return probe.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]


@pytest.mark.parametrize("E,M", [(2, 1), (1, 3), (2, 2)])
def test_epochs_minibatches_equal_composed_steps(E, M):
    """srl_ppo_train_step with E x M updates is bit-identical to E x M srl_ppo_step calls on
    the minibatch row ranges (R-M).  Each update's gradient is held to per-tensor C-T3 against
    the oracle's gradient of that minibatch at the parameters the update started from:
    update 1 on every sample (the fixture is kink-free at theta_0 for the policy clip and the
    value clip); later updates, whose parameters have moved, on the samples the oracle finds
    away from both kinks at those parameters (DESIGN.md §3.3 R-K, §3.5 R-V), through the
    kernel's padding mask.  Value clipping and gradient-norm clipping on: all of NEXT-3 runs."""
    import paper_2306_16688_b200 as P
    from ppo_harness import near_kink, value_kink_free
    cfg = synth.get_config("gfootball").with_(B=20)
    params, b = make_inputs(cfg, seed=13)
    ev = 0.2
    b = value_kink_free(cfg, params, b, ev)
    n = b["n"]
    kw = dict(epochs=E, minibatches=M, value_clip=ev, max_grad_norm=0.05)
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
    u = 0
    for e in range(E):
        for lo, hi in oracle.minibatch_bounds(n, M):
            p0 = c.params().cpu().numpy().astype(np.float64)
            c.step(hi - lo, dv["obs"][lo:hi], dv["actions"][lo:hi], dv["logp_old"][lo:hi],
                   adv[lo:hi], ret[lo:hi], ms, apply=True, v_old=vold[lo:hi])
            ah = (adv[lo:hi].cpu().numpy().astype(np.float64) - mu) / (sd + 1e-8)
            rr, vo = ret[lo:hi].cpu().numpy(), vold[lo:hi].cpu().numpy()
            near = near_kink(cfg, p0, b["obs"][lo:hi], b["actions"][lo:hi], b["logp_old"][lo:hi],
                             v_old=vo, ret=rr, value_clip=ev)
            keep = ~near
            if u == 0:
                assert not near.any()              # the fixture is kink-free at theta_0
                G = c.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
            else:
                assert keep.mean() > 0.9
                G = _probe_grad(cfg, p0, hi - lo, dv["obs"][lo:hi], dv["actions"][lo:hi],
                                dv["logp_old"][lo:hi], adv[lo:hi], ret[lo:hi], ms, vold[lo:hi],
                                keep, value_clip=ev)
            rows = np.flatnonzero(keep)
            g, _, _ = oracle.loss_and_grad(
                cfg.obs_dim, cfg.hidden, cfg.heads, p0, b["obs"][lo:hi][rows],
                b["actions"][lo:hi][rows], b["logp_old"][lo:hi][rows], ah[rows], rr[rows],
                cfg.clip_eps, cfg.value_coef, cfg.entropy_coef, grad_scale=1.0 / (hi - lo),
                v_old=vo[rows], value_clip=ev)
            _check_grads(cfg, G, g)                # per tensor C-T3
            u += 1
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


# ------------------------------------------------------------------ R-T / R-P in the GAE scan
def _flags_tv_valid(rng, T, B):
    u = rng.random((T, B))
    # 1 terminal, 2 time limit, 3 terminal (bit 0 wins), 4 terminal, 6 time limit ((f & 3) == 2)
    f = np.select([u < 0.03, u < 0.06, u < 0.07, u < 0.075, u < 0.08], [1, 2, 3, 4, 6], 0).astype(np.uint8)
    valid = (rng.random((T, B)) < 0.8).astype(np.uint8)
    return f, valid


@pytest.mark.parametrize("T,B", [(7, 33), (128, 96), (400, 50)])
def test_gae_truncation_valid_integer_bit_exact(T, B):
    """gamma = lambda = 1 and small integers (C-B1 style): the truncated bootstrap is exact, so
    adv/ret equal the oracle bit for bit; the masked moments count only valid entries."""
    import paper_2306_16688_b200 as P
    rng = np.random.default_rng(T + B)
    r = rng.integers(-3, 4, (T, B)).astype(np.float32)
    v = rng.integers(-5, 6, (T + 1, B)).astype(np.float32)
    tv = rng.integers(-5, 6, (T, B)).astype(np.float32)
    f, valid = _flags_tv_valid(rng, T, B)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    adv, ret, st = P.gae(dev(r), dev(v), dev(f), 1.0, 1.0, trunc_values=dev(tv), valid=dev(valid))
    ra, rr = oracle.gae(r, v, f, 1.0, 1.0, trunc_values=tv)
    assert np.array_equal(adv.cpu().numpy(), ra.astype(np.float32))
    assert np.array_equal(ret.cpu().numpy(), rr.astype(np.float32))
    st = st.cpu().numpy()
    sel = ra[valid != 0]
    mu, m2 = oracle.moments(sel)
    assert st[0] == sel.size and abs(st[1] - mu) <= 1e-12 * max(1, abs(mu))
    assert abs(st[2] - m2) <= 1e-9 * m2
    # without trunc values a truncation flag is terminal (the core's reading)
    a0, _, _ = P.gae(dev(r), dev(v), dev(f), 1.0, 1.0)
    assert np.array_equal(a0.cpu().numpy(), oracle.gae(r, v, f, 1.0, 1.0)[0].astype(np.float32))


def _padded_inputs(cfg, seed):
    params, b = make_inputs(cfg, seed=seed)
    rng = np.random.default_rng(seed)
    f, valid = _flags_tv_valid(rng, cfg.T, b["Bk"])
    b["dones"] = f
    b["trunc_values"] = rng.normal(size=(cfg.T, b["Bk"])).astype(np.float32)
    b["valid"] = valid
    return params, b


@pytest.mark.parametrize("name", ["gfootball", "hns"])
def test_train_step_truncation_and_padding_parity(name):
    """Whole trainer step with time-limit flags + trunc values and a padding mask: gradient
    (kink-free fixture), statistics and normalisation against the oracle; padding rows
    rewritten with other finite garbage give a bit-identical result (no leak)."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = _padded_inputs(cfg, 17)
    n = b["n"]
    nv = int(b["valid"].sum())
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    assert o["N"] == nv

    def run(bb):
        ctx = _ctx(cfg, params, n)
        d = to_dev(bb)
        tv = torch.from_numpy(bb["trunc_values"]).cuda()
        vm = torch.from_numpy(bb["valid"]).cuda()
        st = P.decode_stats(ctx.train_step(nv, d["rewards"], d["values"], d["dones"], d["obs"],
                                           d["actions"], d["logp_old"], trunc_values=tv, valid=vm))
        return st, ctx.grads().cpu().numpy().astype(np.float64)

    st, G = run(b)
    _check_grads(cfg, G[:cfg.n_params], o["grad"])
    assert st["n_global"] == nv and st["nonfinite"] == 0
    assert abs(st["adv_mean"] - o["mean"]) <= 1e-6 * o["std"]
    assert abs(st["adv_std"] - o["std"]) <= 1e-6 * o["std"]
    assert abs(st["entropy"] - o["sums"][2] / nv) <= TOL * abs(o["sums"][2] / nv)
    g = dict(b)
    pad = b["valid"].reshape(-1) == 0
    g["obs"] = b["obs"].copy()
    g["obs"][pad] = np.float16(3.0)
    g["logp_old"] = b["logp_old"].copy()
    g["logp_old"][pad] = -50.0
    g["actions"] = b["actions"].copy()
    g["actions"][pad] = 0
    st2, G2 = run(g)
    # the pads' activations differ, but every row they feed is multiplied by a zero dZ row
    assert np.array_equal(G2, G)


def test_prefetch_slots_with_truncation_and_padding():
    """NEXT-1 slots carry the optional NEXT-3 arrays: bit-identical to the device path."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("gfootball").with_(B=16)
    params, b = _padded_inputs(cfg, 19)
    nv = int(b["valid"].sum())
    keys = ("rewards", "values", "dones", "obs", "actions", "logp_old", "trunc_values", "valid")
    host = {k: torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys}
    dev = {k: h.cuda() for k, h in host.items()}
    a, c = _ctx(cfg, params, b["n"]), _ctx(cfg, params, b["n"])
    base = [host[k] for k in keys[:6]]
    c.upload(0, *base, trunc_values=host["trunc_values"], valid=host["valid"])
    for k in range(2):
        a.train_step(nv, *[dev[x] for x in keys[:6]], trunc_values=dev["trunc_values"],
                     valid=dev["valid"])
        if k == 0:
            c.upload(1, *base, trunc_values=host["trunc_values"], valid=host["valid"])
        c.train_step_slot(k % 2, nv)
    torch.cuda.synchronize()
    assert torch.equal(a.params(), c.params()) and torch.equal(a.grads(), c.grads())
