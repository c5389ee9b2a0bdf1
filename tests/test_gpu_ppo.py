"""a3-a7 parity: the full trainer step through the C ABI vs the oracle (C-T3..C-T6).

Sizes: every BASELINE.json config at its true T, widths and heads, with B reduced so the
oracle finishes in seconds while still spanning several 128-row tiles and a ragged tail.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import gpu_step, grad_errors, make_inputs, oracle_term_scales

pytestmark = pytest.mark.gpu

REDUCED = {"tiny": 4, "atari": 16, "gfootball": 16, "smac": 20, "hns": 4}
TOL = 2e-3


def _check_grads(cfg, g, gref):
    errs = grad_errors(cfg, g, gref)
    bad = {k: v for k, v in errs.items() if v[0] > TOL or v[1] > TOL}
    assert not bad, bad


def _check_stats(cfg, st, o, sc):
    N = o["N"]
    ref = o["sums"] / N
    assert abs(st["policy_loss"] - ref[0]) <= TOL * sc["pg"]
    assert abs(st["value_loss"] - ref[1]) <= TOL * sc["v"]
    assert abs(st["entropy"] - ref[2]) <= TOL * sc["ent"]
    assert abs(st["clip_fraction"] - ref[3]) <= sc["clip_near"] + 1.0 / N
    assert abs(st["approx_kl"] - ref[4]) <= TOL * sc["kl"]
    assert st["n_global"] == N and st["nonfinite"] == 0


@pytest.mark.parametrize("name", list(REDUCED))
@pytest.mark.parametrize("stress", [False, True])
def test_ppo_step_grad_parity(name, stress):
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=11, stress=stress)
    g = gpu_step(cfg, params, [b], apply=False)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    _check_grads(cfg, g["bucket"][:cfg.n_params], o["grad"])
    _check_stats(cfg, g["stats"], o, oracle_term_scales(cfg, params, [b], o))
    assert abs(g["mean_std"][0] - o["mean"]) <= 1e-6 * o["std"]
    assert abs(g["mean_std"][1] - o["std"]) <= 1e-6 * o["std"]
    assert g["stats"]["step"] == 0          # apply = 0: no Adam, no version bump


@pytest.mark.parametrize("name", ["tiny", "gfootball", "hns"])
def test_ppo_step_apply_adam(name):
    """a6/a7 at K=1: Adam on the kernel's own gradient matches the oracle's Adam on that same
    gradient (C-T5, 'identical G'), t advances, and the fp16 shadow feeds the next forward."""
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=5)
    g = gpu_step(cfg, params, [b], apply=True)
    G = g["bucket"][:cfg.n_params]
    p = params.astype(np.float64).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam(p, m, v, G, 1, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    dp_ref = p - params
    dp = g["params"] - params
    assert np.linalg.norm(dp - dp_ref) / np.linalg.norm(dp_ref) <= 1e-5
    assert np.abs(g["m"] - m).max() <= 1e-6 * np.abs(m).max()
    assert g["stats"]["step"] == 1
    # the step's gradient itself still matches the oracle
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    _check_grads(cfg, G, o["grad"])


def test_two_steps_uses_updated_shadow():
    """Second step's gradient is taken at the Adam-updated parameters (fp16 shadow refreshed)."""
    cfg = synth.get_config("tiny").with_(B=8)
    params, b = make_inputs(cfg, seed=7)
    g = gpu_step(cfg, params, [b], apply=True, n_steps=1)
    p1 = g["params"].astype(np.float32)
    ctx = g["ctx"]
    g2 = gpu_step(cfg, params, [b], apply=False, ctx=ctx)
    o = oracle.ppo_step(cfg, p1, [b], apply=False)
    _check_grads(cfg, g2["bucket"][:cfg.n_params], o["grad"])


@pytest.mark.parametrize("K", [2, 4])
def test_virtual_ranks_equal_full_batch(K):
    """C-T6 on one GPU: K column shards through the same kernels (apply=0, 1/N_global) summed
    in rank order equal the K=1 gradient; both match the oracle's full batch."""
    cfg = synth.get_config("gfootball").with_(B=16)
    params, full = make_inputs(cfg, seed=3)
    shards = [make_inputs(cfg, seed=3, world=K, rank=k)[1] for k in range(K)]
    g1 = gpu_step(cfg, params, [full], apply=False)
    gK = gpu_step(cfg, params, shards, apply=False)
    a, b = gK["bucket"][:cfg.n_params], g1["bucket"][:cfg.n_params]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
    o = oracle.ppo_step(cfg, params, [full], apply=False)
    _check_grads(cfg, a, o["grad"])


@pytest.mark.parametrize("name", ["smac", "hns"])
def test_clip_decisions_differ_only_near_kink(name):
    """Raw recipe (no kink margin): the kernel's clip decisions (fp32 from the fp16 forward)
    may differ from the oracle's (double) only for samples whose oracle log-ratio lies within
    0.01 of a kink; the clip fraction reflects exactly that."""
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=11, margin=0.0)
    g = gpu_step(cfg, params, [b], apply=False)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    xi = oracle.log_pi(cfg, params, b["obs"], b["actions"]) - b["logp_old"]
    near = sum(np.sum(np.abs(xi - np.log(1 + s * cfg.clip_eps)) < 0.01) for s in (1, -1))
    assert abs(g["stats"]["clip_fraction"] - o["sums"][3] / o["N"]) <= near / o["N"] + 1e-7


def test_zero_params_uniform_policy():
    """Zero network: logits 0, entropy = sum ln A_h exactly, V = 0."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("hns").with_(B=4)
    params = np.zeros(cfg.n_params, np.float32)
    _, b = make_inputs(cfg, seed=1)
    g = gpu_step(cfg, params, [b], apply=False)
    assert abs(g["stats"]["entropy"] - sum(np.log(a) for a in cfg.heads)) < 1e-5


def test_nonfinite_skips_adam():
    """A NaN observation makes its loss non-finite: the step reports it and Adam is skipped."""
    cfg = synth.get_config("tiny")
    params, b = make_inputs(cfg, seed=2)
    b["obs"] = b["obs"].copy()
    b["obs"][5, 0] = np.float16(np.nan)
    g = gpu_step(cfg, params, [b], apply=True)
    assert g["stats"]["nonfinite"] >= 1
    assert g["stats"]["step"] == 0
    assert np.array_equal(g["params"], params.astype(np.float64))


@pytest.mark.parametrize("name", ["tiny", "gfootball"])
def test_train_step_equals_composed_calls(name):
    """srl_ppo_train_step (GAE -> norm -> update in one call) is bit-identical to the three
    separate ABI calls, and its GAE / normalisation / gradient match the oracle."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=21)
    g = gpu_step(cfg, params, [b], apply=True)
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
    ctx.load_params(torch.from_numpy(params).cuda())
    d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda()
         for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}
    st = P.decode_stats(ctx.train_step(b["n"], d["rewards"], d["values"], d["dones"], d["obs"],
                                       d["actions"], d["logp_old"]))
    torch.cuda.synchronize()
    p2 = ctx.params().cpu().numpy().astype(np.float64)
    G2 = ctx.grads().cpu().numpy().astype(np.float64)
    assert np.array_equal(p2, g["params"]) and np.array_equal(G2, g["bucket"])
    assert st["step"] == 1
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    _check_grads(cfg, G2[:cfg.n_params], o["grad"])
    assert abs(st["adv_mean"] - o["mean"]) <= 1e-6 * o["std"]
    assert abs(st["adv_std"] - o["std"]) <= 1e-6 * o["std"]


def test_prefetch_slots_equal_device_path():
    """NEXT-1 (§4.1): host batches uploaded into alternating device slots on the
    context's copy stream give bit-identical results to steps on device-resident inputs."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("gfootball").with_(B=16)
    params, b = make_inputs(cfg, seed=8)
    keys = ("rewards", "values", "dones", "obs", "actions", "logp_old")
    host = [torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys]
    dev = [h.cuda() for h in host]
    spec = P.NetSpec.from_config(cfg)
    a = P.PPOContext(spec, max_local_n=b["n"])
    c = P.PPOContext(spec, max_local_n=b["n"])
    for ctx in (a, c):
        ctx.load_params(torch.from_numpy(params).cuda())
    c.upload(0, *host)
    for k in range(3):
        a.train_step(b["n"], *dev)
        if k + 1 < 3:
            c.upload((k + 1) % 2, *host)
        st = P.decode_stats(c.train_step_slot(k % 2, b["n"]))
    torch.cuda.synchronize()
    assert st["step"] == 3
    assert torch.equal(a.params(), c.params()) and torch.equal(a.grads(), c.grads())
    with pytest.raises(P.SrlError):
        c.train_step_slot(0, b["n"])          # consumed: nothing uploaded into slot 0 since


def test_prefetch_slots_against_oracle():
    """NEXT-1 slot path (host batch -> device slot on the copy stream -> train step) checked
    against the ORACLE at every one of 3 chained steps, not against the device path:
    step k's gradient vs the oracle's gradient of the batch at the parameters step k started
    from (C-T3; from step 2 on over the samples the oracle finds away from the clip kinks at
    those parameters, through the padding mask), and step k's parameter / Adam-moment update
    vs the oracle's Adam (C-6) applied to that same gradient with the moments carried in
    double from step 1 (C-T5, 'identical G')."""
    import paper_2306_16688_b200 as P
    from ppo_harness import near_kink
    cfg = synth.get_config("gfootball").with_(B=16)
    params, b = make_inputs(cfg, seed=8)
    n = b["n"]
    keys = ("rewards", "values", "dones", "obs", "actions", "logp_old")
    host = [torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys]
    spec = P.NetSpec.from_config(cfg)
    c = P.PPOContext(spec, max_local_n=n)
    c.load_params(torch.from_numpy(params).cuda())
    o0 = oracle.ppo_step(cfg, params, [b], apply=False)
    ahat = (o0["adv"][0] - o0["mean"]) / (o0["std"] + 1e-8)
    m = np.zeros(cfg.n_params)
    v = np.zeros(cfg.n_params)
    c.upload(0, *host)
    for k in range(3):
        p_k = c.params().cpu().numpy().astype(np.float64)
        if k + 1 < 3:
            c.upload((k + 1) % 2, *host)
        st = P.decode_stats(c.train_step_slot(k % 2, n))
        torch.cuda.synchronize()
        G = c.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
        near = near_kink(cfg, p_k, b["obs"], b["actions"], b["logp_old"])
        if k == 0:
            assert not near.any()
            Gk = G
        else:
            assert near.mean() < 0.05
            probe = P.PPOContext(spec, max_local_n=n)
            probe.load_params(torch.from_numpy(p_k.astype(np.float32)).cuda())
            d = {kk: torch.from_numpy(np.ascontiguousarray(b[kk])).cuda() for kk in keys}
            adv, ret, gst = P.gae(d["rewards"], d["values"], d["dones"], cfg.gamma, cfg.lam)
            ms = P.adv_norm(adv.reshape(-1), local_stats=gst)
            probe.step(n, d["obs"], d["actions"], d["logp_old"], adv.reshape(-1), ret.reshape(-1), ms,
                       apply=False, valid=torch.from_numpy((~near).astype(np.uint8)).cuda())
            Gk = probe.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
        rows = np.flatnonzero(~near)
        g, _, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, p_k, b["obs"][rows],
                                       b["actions"][rows], b["logp_old"][rows], ahat[rows],
                                       o0["ret"][0][rows], cfg.clip_eps, cfg.value_coef,
                                       cfg.entropy_coef, grad_scale=1.0 / n)
        _check_grads(cfg, Gk, g)
        p_ref = p_k.copy()
        oracle.adam(p_ref, m, v, G, k + 1, cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
        p_next = c.params().cpu().numpy().astype(np.float64)
        assert np.linalg.norm((p_next - p_k) - (p_ref - p_k)) <= 1e-5 * np.linalg.norm(p_ref - p_k)
        mg = c.adam_state()[0].cpu().numpy().astype(np.float64)
        assert np.abs(mg - m).max() <= 1e-6 * np.abs(m).max()
        assert st["step"] == k + 1


@pytest.mark.parametrize("name", ["atari", "gfootball", "hns"])
def test_step_is_deterministic(name):
    """Two contexts, same inputs, two chained steps each: bit-identical gradients, parameters
    and Adam moments (fixed-order split/partial sums in the fused update kernel, no atomics
    on floating-point values)."""
    cfg = synth.get_config(name).with_(B=REDUCED[name] * synth.get_config(name).agents)
    params, b = make_inputs(cfg, seed=23)
    outs = []
    for _ in range(2):
        g = gpu_step(cfg, params, [b], apply=True, n_steps=2)
        outs.append(g)
    for k in ("bucket", "params", "m", "v"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
