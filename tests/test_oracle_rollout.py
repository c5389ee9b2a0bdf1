"""Pins for the oracle's NEXT-2 policy-worker inference (reading R-S):
the counter RNG against SplitMix64's published outputs, deterministic mode against numpy's
argmax of the forward, and sampled frequencies against the softmax probabilities."""
import numpy as np

import oracle

M64 = (1 << 64) - 1


def _sm64(x):
    """Test-side SplitMix64 step (state x -> output for state x + golden gamma)."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_splitmix64_published_sequence_and_uniform():
    # SplitMix64 seeded with 0: 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f
    g = 0x9E3779B97F4A7C15
    assert [_sm64(0), _sm64(g), _sm64(2 * g & M64)] == [
        0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    rng = np.random.default_rng(0)
    for _ in range(50):
        seed, key = int(rng.integers(0, 1 << 62)), int(rng.integers(0, 1 << 62))
        h = int(rng.integers(0, 8))
        want = (_sm64((_sm64(seed ^ key) + h) & M64) >> 40) / float(1 << 24)
        assert oracle.uniform(seed, key, h) == want
    u = np.array([oracle.uniform(7, k, 0) for k in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01


def _net(seed, obs_dim=6, hidden=(16, 8), heads=(5, 3)):
    P = oracle.param_count(obs_dim, hidden, heads)
    p = np.random.default_rng(seed).uniform(-0.8, 0.8, P)
    return (obs_dim, hidden, heads), p


def test_deterministic_is_argmax_of_forward():
    net, p = _net(1)
    obs = np.random.default_rng(1).normal(size=(200, net[0]))
    act, lp, val, _ = oracle.rollout(*net, p, obs, deterministic=True)
    z = oracle.forward(*net, p, obs)
    np.testing.assert_array_equal(act[:, 0], np.argmax(z[:, :5], axis=1))
    np.testing.assert_array_equal(act[:, 1], np.argmax(z[:, 5:8], axis=1))
    cls = type("c", (), dict(obs_dim=net[0], hidden=net[1], heads=net[2]))
    np.testing.assert_allclose(lp, oracle.log_pi(cls(), p, obs, act), rtol=0, atol=1e-13)
    np.testing.assert_array_equal(val, z[:, -1])


def test_sampled_frequencies_match_softmax():
    """One observation, 120k request keys: per-head action counts against the softmax
    probabilities (chi-square, 6 sigma); an off-by-one in the inverse CDF shifts them."""
    net, p = _net(2)
    x = np.random.default_rng(2).normal(size=(1, net[0]))
    n = 120_000
    act, lp, _, _ = oracle.rollout(*net, p, np.repeat(x, n, 0), seed=11,
                                   keys=np.arange(n, dtype=np.uint64) * 7919)
    z = oracle.forward(*net, p, x)[0]
    s = 0
    for h, a in enumerate(net[2]):
        pr = np.exp(z[s:s + a] - z[s:s + a].max())
        pr /= pr.sum()
        cnt = np.bincount(act[:, h], minlength=a)
        chi2 = np.sum((cnt - n * pr) ** 2 / (n * pr))
        assert chi2 < a - 1 + 6 * np.sqrt(2 * (a - 1)), (h, chi2)
        s += a
    # logp is log pi of the sampled actions
    cls = type("c", (), dict(obs_dim=net[0], hidden=net[1], heads=net[2]))
    np.testing.assert_allclose(lp[:50], oracle.log_pi(cls(), p, np.repeat(x, 50, 0), act[:50]),
                               rtol=0, atol=1e-13)


def test_same_key_same_action_and_key_default():
    net, p = _net(3)
    obs = np.random.default_rng(3).normal(size=(64, net[0]))
    a1 = oracle.rollout(*net, p, obs, seed=5)[0]
    a2 = oracle.rollout(*net, p, obs, seed=5, keys=np.arange(64, dtype=np.uint64))[0]
    a3 = oracle.rollout(*net, p, obs, seed=6)[0]
    assert np.array_equal(a1, a2) and not np.array_equal(a1, a3)
