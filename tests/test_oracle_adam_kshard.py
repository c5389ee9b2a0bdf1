"""Pins for oracle C-5 (K-shard sum) and C-6 (Adam)."""
import numpy as np
import pytest

import oracle
import synth
from ppo_harness import make_inputs


def test_adam_step1_closed_form():
    """Step 1: m_hat = g, v_hat = g^2, so dp = -lr g / (|g| + eps)."""
    rng = np.random.default_rng(0)
    g = rng.normal(size=100) * 10.0 ** rng.integers(-6, 2, 100)
    p = rng.normal(size=100)
    p0 = p.copy()
    m, v = np.zeros(100), np.zeros(100)
    oracle.adam(p, m, v, g, 1, lr=3e-4)
    np.testing.assert_allclose(p - p0, -3e-4 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=1e-20)


def test_adam_matches_torch_optim_double():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    p = rng.normal(size=50)
    m, v = np.zeros(50), np.zeros(50)
    tp = torch.tensor(p.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([tp], lr=3e-4, betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 5):
        g = rng.normal(size=50)
        oracle.adam(p, m, v, g, t)
        tp.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
    np.testing.assert_allclose(p, tp.detach().numpy(), rtol=0, atol=1e-15)


def _with_logp(cfg, params, sh):
    sh["logp_old"] = oracle.log_pi(cfg, params, sh["obs"], sh["actions"]) - sh["xi"]
    return sh


@pytest.mark.parametrize("K", [2, 4])
def test_kshard_equals_full_batch(K):
    """K shards with per-shard grads scaled by 1/N_global, summed in rank order,
    equal the K=1 full-batch gradient (<=1e-12 relative, double)."""
    cfg = synth.get_config("tiny").with_(B=8)
    params = synth.make_params(cfg, 0)
    full = _with_logp(cfg, params, synth.make_batch(cfg, seed=1))
    shards = [_with_logp(cfg, params, synth.make_batch(cfg, seed=1, world=K, rank=k))
              for k in range(K)]
    # shards concatenate to the full batch (same counters)
    T = cfg.T
    np.testing.assert_array_equal(np.concatenate([s["rewards"] for s in shards], 1), full["rewards"])
    o1 = oracle.ppo_step(cfg, params, [full], apply=False)
    oK = oracle.ppo_step(cfg, params, shards, apply=False)
    assert abs(o1["mean"] - oK["mean"]) < 1e-14 and abs(o1["std"] - oK["std"]) < 1e-14
    rel = np.linalg.norm(oK["grad"] - o1["grad"]) / np.linalg.norm(o1["grad"])
    assert rel <= 1e-12
    np.testing.assert_allclose(oK["sums"], o1["sums"], rtol=1e-12, atol=1e-13)
    # the GAE outputs of the shards are the column blocks of the full output
    fa = o1["adv"][0].reshape(T, cfg.B)
    c = 0
    for s, a in zip(shards, oK["adv"]):
        np.testing.assert_array_equal(a.reshape(T, s["Bk"]), fa[:, c:c + s["Bk"]])
        c += s["Bk"]


def test_kshard_opposite_grads_cancel():
    """members with gradients g and -g reduce to zero (sum in rank order)."""
    rng = np.random.default_rng(3)
    g = rng.normal(size=1000)
    assert np.array_equal(g + (-g), np.zeros_like(g))


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_all_core_driver_equals_single_thread(threads):
    """bench.py's all-core cpu_baseline driver (oracle_loss_and_grad_mt) computes the same
    gradient and loss sums as oracle_loss_and_grad, up to the order of the block sums."""
    cfg = synth.get_config("gfootball").with_(B=24)            # 4800 rows: the driver path
    params, b = make_inputs(cfg, seed=2)
    o1 = oracle.ppo_step(cfg, params, [b], apply=True, threads=1)
    oT = oracle.ppo_step(cfg, params, [b], apply=True, threads=threads)
    assert np.linalg.norm(oT["grad"] - o1["grad"]) <= 1e-12 * np.linalg.norm(o1["grad"])
    assert np.allclose(oT["sums"], o1["sums"], rtol=1e-12, atol=1e-12)
    assert np.linalg.norm(oT["params"] - o1["params"]) <= 1e-12 * np.linalg.norm(o1["params"])
