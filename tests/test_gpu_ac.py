"""NEXT-3 remainder: separate actor and critic trunks (srl_ppo_config.separate_critic; SURVEY.md
§8(f) NEXT-3; DESIGN.md §3.5 reading R-AC) through the C ABI against the
two-trunk oracle (tests/test_oracle_ac.py pins it): gradients per tensor at C-T3, loss terms
at C-T4, Adam on the kernel's own gradient, the second step at the updated parameters (fp16
shadows and the head-bias mirror refreshed by Adam), deterministic-mode inference, and the
tied-trunk identity against the shared-trunk context."""
import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import gpu_step, grad_errors, make_inputs, oracle_term_scales

pytestmark = pytest.mark.gpu

TOL = 2e-3
REDUCED = {"tiny": 4, "atari": 8, "gfootball": 16, "smac": 10, "hns": 4}


def _cfg(name):
    base = synth.get_config(name)
    return base.with_(B=REDUCED[name] * base.agents, separate_critic=True)


def _check_grads(cfg, g, gref, tol=TOL):
    errs = grad_errors(cfg, g, gref)
    bad = {k: v for k, v in errs.items() if v[0] > tol or v[1] > tol}
    assert not bad, bad


@pytest.mark.parametrize("name", list(REDUCED))
def test_ac_grad_parity(name):
    cfg = _cfg(name)
    params, b = make_inputs(cfg, seed=51)
    g = gpu_step(cfg, params, [b], apply=False)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    _check_grads(cfg, g["bucket"][:cfg.n_params], o["grad"])
    sc = oracle_term_scales(cfg, params, [b], o)
    st, N = g["stats"], o["N"]
    ref = o["sums"] / N
    assert abs(st["policy_loss"] - ref[0]) <= TOL * sc["pg"]
    assert abs(st["value_loss"] - ref[1]) <= TOL * sc["v"]
    assert abs(st["entropy"] - ref[2]) <= TOL * sc["ent"]
    assert st["n_global"] == N and st["nonfinite"] == 0


@pytest.mark.parametrize("name", ["tiny", "gfootball", "hns"])
def test_ac_adam_and_second_step(name):
    cfg = _cfg(name)
    params, b = make_inputs(cfg, seed=53)
    g = gpu_step(cfg, params, [b], apply=True)
    G = g["bucket"][:cfg.n_params]
    p = params.astype(np.float64).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam(p, m, v, G, 1, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    dp = g["params"] - params
    assert np.linalg.norm(dp - (p - params)) <= 1e-5 * np.linalg.norm(p - params)
    assert g["stats"]["step"] == 1
    # the second step's gradient is taken at the updated parameters: weights through the fp16
    # shadows, the two head biases through the contiguous fp32 mirror.  At those parameters
    # some samples may sit on a clip kink (DESIGN.md §3.3 R-K): they are left out of the
    # comparison through the kernel's padding mask (R-P)
    import paper_2306_16688_b200 as P
    from ppo_harness import near_kink
    p1 = g["params"].astype(np.float32)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    keep = ~near_kink(cfg, p1.astype(np.float64), b["obs"], b["actions"], b["logp_old"])
    assert keep.mean() > 0.95
    d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda() for k in ("obs", "actions", "logp_old")}
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    ctx = g["ctx"]
    n = b["n"]
    ms = torch.tensor([o["mean"], o["std"]], dtype=torch.float64, device="cuda")
    ctx.step(n, d["obs"], d["actions"], d["logp_old"], t(o["adv"][0]), t(o["ret"][0]), ms,
             apply=False, valid=torch.from_numpy(keep.astype(np.uint8)).cuda())
    G2 = ctx.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
    rows = np.flatnonzero(keep)
    ahat = (o["adv"][0] - o["mean"]) / (o["std"] + 1e-8)
    g2, _, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, p1.astype(np.float64),
                                    b["obs"][rows], b["actions"][rows], b["logp_old"][rows],
                                    ahat[rows], o["ret"][0][rows], cfg.clip_eps, cfg.value_coef,
                                    cfg.entropy_coef, grad_scale=1.0 / n, separate=True)
    _check_grads(cfg, G2, g2)


def test_ac_tied_trunks_equal_shared_context():
    """A two-trunk context whose trunks hold the same parameters computes the shared net:
    the shared context's trunk gradient = actor + critic trunk gradients, head rows equal."""
    import paper_2306_16688_b200 as P
    base = synth.get_config("gfootball").with_(B=16)
    cfg = base.with_(separate_critic=True)
    ps, b = make_inputs(base, seed=55)
    d = base.dims
    L = len(base.hidden)
    T = sum(d[i + 1] * d[i] + d[i + 1] for i in range(L))
    A, h = base.n_actions, d[L]
    trunk, head = ps[:T], ps[T:]
    Wh, bh = head[:(A + 1) * h].reshape(A + 1, h), head[(A + 1) * h:]
    pac = np.concatenate([trunk, Wh[:A].ravel(), bh[:A], trunk, Wh[A:].ravel(), bh[A:]]).astype(np.float32)
    gs = gpu_step(base, ps, [b], apply=False)["bucket"]
    ga = gpu_step(cfg, pac, [b], apply=False)["bucket"]
    Gs = gs[:base.n_params]
    Ga = ga[:cfg.n_params]
    o_pi, o_c = T, T + A * h + A
    o_v = o_c + T
    # the two paths sum their fp32 partials in different orders (other split counts): the
    # identity holds to fp32 summation error, far below the 2e-3 parity tolerance
    scale = np.abs(Gs).max() * 10
    assert np.abs((Ga[:T] + Ga[o_c:o_v]) - Gs[:T]).max() <= 1e-5 * scale
    assert np.abs(Ga[o_pi:o_c] - np.concatenate([Gs[T:T + A * h], Gs[T + (A + 1) * h:T + (A + 1) * h + A]])).max() <= 1e-5 * scale
    assert np.abs(Ga[o_v:] - np.concatenate([Gs[T + A * h:T + (A + 1) * h], Gs[-1:]])).max() <= 1e-5 * scale


def test_ac_rollout_deterministic():
    """NEXT-2 inference on a two-trunk context: argmax actions, log-probs and values equal the
    two-trunk oracle forward where the oracle's top-2 logit gap exceeds 5e-3."""
    import paper_2306_16688_b200 as P
    cfg = _cfg("atari")
    params, b = make_inputs(cfg, seed=57)
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
    ctx.load_params(torch.from_numpy(params).cuda())
    obs = torch.from_numpy(b["obs"]).cuda()
    act, lp, val = ctx.rollout(obs, deterministic=True)
    torch.cuda.synchronize()
    z = oracle.forward(cfg.obs_dim, cfg.hidden, cfg.heads, params, b["obs"], separate=True)
    logits = z[:, :-1]
    top2 = np.sort(logits, axis=1)[:, -2:]
    safe = (top2[:, 1] - top2[:, 0]) > 5e-3
    assert safe.mean() > 0.9
    assert np.array_equal(act.cpu().numpy()[safe, 0], logits.argmax(1)[safe])
    assert np.max(np.abs(val.cpu().numpy() - z[:, -1])) <= 2e-3 * (1 + np.abs(z[:, -1]).mean())
