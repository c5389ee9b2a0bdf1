"""Pins for the oracle's NEXT-3 PPO variants:
value-loss clipping (reading R-V), global gradient-norm clipping (R-G) and
epochs x minibatches (R-M).

Against: hand-derived single-sample values, central finite differences of the clipped
loss, torch.nn.utils.clip_grad_norm_ (library routine), and the linearity invariant
sum_k (N_k / N) g_k = g_full of minibatch gradients taken at fixed parameters.
"""
import math

import numpy as np
import pytest

import oracle
import synth


def _one(v_old, ret, value_clip, cv=0.5):
    """Zero network (V = 0, uniform logits), one sample, A_hat = 0, grad_scale = 1."""
    net = (2, (), (3,))
    P = oracle.param_count(*net)
    g, sums, ps = oracle.loss_and_grad(*net, np.zeros(P), np.array([[0.3, -0.7]]),
                                       np.array([[1]], np.int32), np.zeros(1), np.zeros(1),
                                       np.array([ret]), 0.2, cv, 0.0, grad_scale=1.0,
                                       want_per_sample=True, v_old=np.array([v_old]),
                                       value_clip=value_clip)
    # layout: W[4][2] then b[4]; the value output is row 3
    return g[6:8], g[11], sums[1], ps[0]


def test_value_clip_hand_cases():
    """V = 0.  (a) v_old = 1, R = -0.5, eps_v = 0.2: V_c = 0.8, (V-R)^2 = 0.25 <
    (V_c-R)^2 = 1.69 -> l_v = 1.69 and no gradient (V outside the clip band).
    (b) v_old = 1, R = 2: (V-R)^2 = 4 > (V_c-R)^2 = 1.44 -> unclipped: dl/db_V = c_v * 2(0-2) = -2.
    (c) v_old = 0.1, R = 1: |V - v_old| = 0.1 <= 0.2 -> V_c = V, l_v = 1, db_V = -1."""
    gw, gb, l, loss = _one(1.0, -0.5, 0.2)
    assert abs(l - 1.69) < 1e-15 and abs(loss - 0.5 * 1.69) < 1e-15
    assert gb == 0.0 and np.all(gw == 0.0)
    gw, gb, l, _ = _one(1.0, 2.0, 0.2)
    assert l == 4.0 and gb == -2.0
    np.testing.assert_allclose(gw, -2.0 * np.array([0.3, -0.7]), rtol=0, atol=1e-15)
    gw, gb, l, _ = _one(0.1, 1.0, 0.2)
    assert l == 1.0 and gb == -1.0
    # value_clip <= 0 or v_old absent: plain squared error
    assert _one(1.0, -0.5, 0.0)[2] == 0.25


def test_value_clip_huge_band_is_unclipped():
    net = (4, (8,), (3, 2))
    P = oracle.param_count(*net)
    rng = np.random.default_rng(0)
    p = rng.uniform(-0.5, 0.5, P)
    n = 9
    obs = rng.normal(size=(n, 4))
    act = np.stack([rng.integers(0, 3, n), rng.integers(0, 2, n)], 1).astype(np.int32)
    args = (rng.normal(size=n), rng.normal(size=n), rng.normal(size=n))
    g0, s0, _ = oracle.loss_and_grad(*net, p, obs, act, *args)
    g1, s1, _ = oracle.loss_and_grad(*net, p, obs, act, *args, v_old=rng.normal(size=n),
                                     value_clip=1e9)
    assert np.array_equal(g0, g1) and np.array_equal(s0, s1)


def test_value_clip_finite_difference():
    """Central FD (step 1e-5) of the mean clipped loss; the fixture keeps every sample at
    least 0.05 from the band edges |V - v_old| = eps_v and |l_c - l_v| >= 0.01 (kink-free)."""
    net = (4, (6, 5), (3,))
    P = oracle.param_count(*net)
    rng = np.random.default_rng(7)
    p = rng.uniform(-1, 1, P) * 0.6
    n = 16
    obs = rng.normal(size=(n, 4))
    act = rng.integers(0, 3, (n, 1)).astype(np.int32)
    V = oracle.forward(*net, p, obs)[:, -1]
    ev = 0.2
    delta = np.array([0.05, -0.05, 0.5, -0.5] * 4)           # inside / outside the band
    vold = V - delta
    ret = rng.normal(size=n) * 0.8
    Vc = vold + np.clip(V - vold, -ev, ev)
    for i in range(n):              # outside the band keep |l_c - l_v| >= 0.01 (inside: V_c = V)
        while abs(delta[i]) > ev and abs((Vc[i] - ret[i]) ** 2 - (V[i] - ret[i]) ** 2) < 0.01:
            ret[i] += 0.1
    lc, lv = (Vc - ret) ** 2, (V - ret) ** 2
    assert (lc > lv).sum() >= 3 and (lc < lv).sum() >= 3     # both branches exercised
    lo, ah = rng.normal(size=n) * 0.1, rng.normal(size=n)
    kw = dict(clip_eps=10.0, value_coef=0.5, entropy_coef=0.01, v_old=vold, value_clip=ev)
    grad, _, _ = oracle.loss_and_grad(*net, p, obs, act, lo, ah, ret, **kw)

    def total(pp):
        _, _, ps = oracle.loss_and_grad(*net, pp, obs, act, lo, ah, ret, want_per_sample=True, **kw)
        return ps.mean()

    h = 1e-5
    fd = np.empty(P)
    for k in range(P):
        pp, pm = p.copy(), p.copy()
        pp[k] += h
        pm[k] -= h
        fd[k] = (total(pp) - total(pm)) / (2 * h)
    err = np.abs(grad - fd)
    assert np.all(err <= 1e-6 * np.maximum(np.abs(fd), np.abs(fd).max() * 1e-3))


@pytest.mark.parametrize("max_norm", [0.5, 3.0, 100.0])
def test_clip_grad_norm_matches_torch(max_norm):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(int(max_norm * 10))
    g = rng.normal(size=257) * 0.4
    ref = torch.nn.Parameter(torch.zeros(257, dtype=torch.float64))
    ref.grad = torch.tensor(g.copy())
    tn = float(torch.nn.utils.clip_grad_norm_([ref], max_norm))
    ours = g.copy()
    norm = oracle.clip_grad_norm(ours, max_norm)
    assert abs(norm - tn) <= 1e-13 * tn
    np.testing.assert_allclose(ours, ref.grad.numpy(), rtol=1e-15, atol=0)
    assert np.linalg.norm(ours) <= max_norm * (1 + 1e-12)
    # idempotent up to the 1e-6 guard
    again = ours.copy()
    oracle.clip_grad_norm(again, max_norm)
    np.testing.assert_allclose(again, ours, rtol=4e-6 / max_norm, atol=0)


def _with_logp(cfg, params, sh):
    sh["logp_old"] = oracle.log_pi(cfg, params, sh["obs"], sh["actions"]) - sh["xi"]
    return sh


@pytest.mark.parametrize("K,M", [(1, 3), (2, 2)])
def test_minibatch_gradients_average_to_full_batch(K, M):
    """At fixed parameters (apply=False) the minibatch gradients, weighted by N_k / N, sum to
    the full-batch gradient and the loss sums add up (linearity of the mean loss); a second
    epoch repeats the first exactly."""
    cfg = synth.get_config("tiny").with_(B=12)
    params = synth.make_params(cfg, 0)
    shards = [_with_logp(cfg, params, synth.make_batch(cfg, seed=2, world=K, rank=k))
              for k in range(K)]
    full = oracle.ppo_step(cfg, params, shards, apply=False)
    mb = oracle.ppo_step(cfg, params, shards, apply=False, minibatches=M, epochs=2)
    assert len(mb["grads"]) == 2 * M
    n_loc = [s["n"] for s in shards]
    Nk = [sum(b[k][1] - b[k][0] for b in (oracle.minibatch_bounds(n, M) for n in n_loc))
          for k in range(M)]
    assert sum(Nk) == full["N"]
    avg = sum(Nk[k] / full["N"] * mb["grads"][k] for k in range(M))
    assert np.linalg.norm(avg - full["grad"]) <= 1e-12 * np.linalg.norm(full["grad"])
    np.testing.assert_allclose(sum(mb["sums_all"][:M]), full["sums"], rtol=1e-12, atol=1e-12)
    for k in range(M):
        assert np.array_equal(mb["grads"][k], mb["grads"][M + k])


def test_grad_norm_clip_in_step_and_adam_count():
    """max_grad_norm below the gradient norm: the clipped gradient has exactly that norm
    (to the 1e-6 guard) and each of the E*M updates advances the Adam step."""
    cfg = synth.get_config("tiny").with_(B=8)
    params = synth.make_params(cfg, 1)
    sh = [_with_logp(cfg, params, synth.make_batch(cfg, seed=3))]
    o = oracle.ppo_step(cfg, params, sh, apply=False)
    n0 = float(np.linalg.norm(o["grad"]))
    oc = oracle.ppo_step(cfg, params, sh, apply=False, max_grad_norm=0.5 * n0)
    assert abs(oc["grad_norm"] - n0) <= 1e-12 * n0
    assert abs(np.linalg.norm(oc["grad"]) - 0.5 * n0) <= 1e-6 * n0
    np.testing.assert_allclose(oc["grad"], o["grad"] * (0.5 * n0 / (n0 + 1e-6)), rtol=1e-14)
    # E*M updates == the same number of single-update calls chained by hand
    a = oracle.ppo_step(cfg, params, sh, epochs=2, minibatches=1)
    b1 = oracle.ppo_step(cfg, params, sh)
    b2 = oracle.ppo_step(cfg, b1["params"], sh, adam_state=(b1["m"], b1["v"]), t=2)
    assert np.array_equal(a["params"], b2["params"])
    assert not math.isclose(float(np.abs(a["params"] - b1["params"]).max()), 0.0)


# ------------------------------------------------------------------ R-T: time-limit truncation
def test_truncation_hand_case():
    """One column, gamma = 0.5, lambda = 1, flags [0, 2, 0] (bit 1 = time limit at t = 1),
    trunc value 7 at t = 1:  t=2: delta = 3 + 0.5*2 - 1.5 = 2.5 = A_2;  t=1: delta = 2 +
    0.5*7 - 1 = 4.5 and the chain is cut: A_1 = 4.5;  t=0: delta = 1 + 0.5*1 - 0.5 = 1,
    A_0 = 1 + 0.5*4.5 = 3.25.  Without trunc_values the flag is terminal: A_1 = 2 - 1 = 1."""
    r = np.array([[1.0], [2.0], [3.0]], np.float32)
    v = np.array([[0.5], [1.0], [1.5], [2.0]], np.float32)
    f = np.array([[0], [2], [0]], np.uint8)
    tv = np.array([[0.0], [7.0], [0.0]], np.float32)
    a, ret = oracle.gae(r, v, f, 0.5, 1.0, trunc_values=tv)
    assert a[:, 0].tolist() == [3.25, 4.5, 2.5]
    assert ret[:, 0].tolist() == [3.75, 5.5, 4.0]
    a0, _ = oracle.gae(r, v, f, 0.5, 1.0)
    assert a0[:, 0].tolist() == [1.0 + 0.5 * 1.0, 1.0, 2.5]
    # a terminal flag (bit 0) wins over a truncation bit
    a3, _ = oracle.gae(r, v, np.array([[0], [3], [0]], np.uint8), 0.5, 1.0, trunc_values=tv)
    assert a3[1, 0] == 1.0
    # only (flag & 3) == 2 is a time limit (DESIGN.md §3.5 R-T): 0x04 is terminal, 0x06 truncates
    a4, _ = oracle.gae(r, v, np.array([[0], [4], [0]], np.uint8), 0.5, 1.0, trunc_values=tv)
    assert a4[1, 0] == 1.0
    a6, _ = oracle.gae(r, v, np.array([[0], [6], [0]], np.uint8), 0.5, 1.0, trunc_values=tv)
    assert a6[:, 0].tolist() == [3.25, 4.5, 2.5]


def test_truncation_equals_split_column_with_bootstrap():
    """A column truncated at t equals, on rows 0..t, the un-flagged prefix column whose
    bootstrap row is the truncated state's value (bit-exact: same double operations)."""
    rng = np.random.default_rng(5)
    T = 12
    r = rng.normal(size=(T, 1)).astype(np.float32)
    v = rng.normal(size=(T + 1, 1)).astype(np.float32)
    f = np.zeros((T, 1), np.uint8)
    t = 6
    f[t, 0] = 2
    tv = rng.normal(size=(T, 1)).astype(np.float32)
    a, _ = oracle.gae(r, v, f, 0.99, 0.95, trunc_values=tv)
    vp = np.concatenate([v[:t + 1], tv[t:t + 1]])
    ap, _ = oracle.gae(r[:t + 1], vp, np.zeros((t + 1, 1), np.uint8), 0.99, 0.95)
    assert np.array_equal(a[:t + 1], ap)
    # and the rows after the cut are the GAE of the suffix on its own
    As, _ = oracle.gae(r[t + 1:], v[t + 1:], f[t + 1:], 0.99, 0.95)
    assert np.array_equal(a[t + 1:], As)


# ------------------------------------------------------------------ R-P: padding mask
def _padded_shard(cfg, params, seed):
    b = synth.make_batch(cfg, seed=seed)
    b["logp_old"] = oracle.log_pi(cfg, params, b["obs"], b["actions"]) - b["xi"]
    rng = np.random.default_rng(seed)
    valid = (rng.random((cfg.T, b["Bk"])) < 0.7).astype(np.uint8)
    valid[0, 0] = 1
    b["valid"] = valid
    return b


def test_valid_mask_moments_and_all_ones():
    cfg = synth.get_config("tiny").with_(B=8)
    params = synth.make_params(cfg, 2)
    b = _padded_shard(cfg, params, 6)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    a = o["adv"][0][b["valid"].reshape(-1) != 0]
    assert o["N"] == int(b["valid"].sum())
    assert abs(o["mean"] - a.mean()) <= 1e-14 * max(1.0, abs(a.mean()))     # numpy moments
    assert abs(o["std"] - a.std()) <= 1e-13 * a.std()
    ones = dict(b, valid=np.ones_like(b["valid"]))
    plain = {k: v for k, v in b.items() if k != "valid"}
    o1, o2 = oracle.ppo_step(cfg, params, [ones], apply=False), oracle.ppo_step(cfg, params, [plain], apply=False)
    assert np.array_equal(o1["grad"], o2["grad"]) and o1["N"] == o2["N"]


def test_valid_mask_padding_never_leaks():
    """Garbage (NaN observations, out-of-range log-probs, other actions) in padding rows
    leaves every output unchanged."""
    cfg = synth.get_config("tiny").with_(B=8)
    params = synth.make_params(cfg, 3)
    b = _padded_shard(cfg, params, 7)
    o = oracle.ppo_step(cfg, params, [b], apply=True)
    pad = b["valid"].reshape(-1) == 0
    g = dict(b)
    g["obs"] = b["obs"].copy()
    g["obs"][pad] = np.float16(np.nan)
    g["logp_old"] = b["logp_old"].copy()
    g["logp_old"][pad] = 1e6
    g["actions"] = b["actions"].copy()
    g["actions"][pad] = 0
    og = oracle.ppo_step(cfg, params, [g], apply=True)
    assert np.array_equal(o["grad"], og["grad"]) and np.array_equal(o["params"], og["params"])
    assert np.array_equal(o["sums"], og["sums"])
