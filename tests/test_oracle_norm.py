"""Pins for oracle C-2 (advantage normalisation, C-A4)."""
import numpy as np

import oracle


def test_moments_match_library():
    rng = np.random.default_rng(0)
    a = rng.normal(3.0, 2.0, 10001)
    mu, m2 = oracle.moments(a)
    assert abs(mu - np.mean(a)) <= 1e-13 * abs(np.mean(a))
    assert abs(m2 / a.size - np.var(a)) <= 1e-12 * np.var(a)


def test_normalised_mean_zero_std_one():
    rng = np.random.default_rng(1)
    a = rng.normal(-7.0, 0.3, 5000)
    out, mu, sd = oracle.adv_norm(a, eps=1e-8)
    assert abs(out.mean()) < 1e-12
    assert abs(out.std() - sd / (sd + 1e-8)) < 1e-12


def test_affine_invariance():
    rng = np.random.default_rng(2)
    a = rng.normal(size=777)
    o1, _, _ = oracle.adv_norm(a, eps=0.0)
    o2, _, _ = oracle.adv_norm(4.5 * a - 11.0, eps=0.0)
    np.testing.assert_allclose(o1, o2, rtol=0, atol=1e-12)


def test_unbiased_flag():
    rng = np.random.default_rng(3)
    a = rng.normal(size=32)
    _, _, s_pop = oracle.adv_norm(a, unbiased=False)
    _, _, s_unb = oracle.adv_norm(a, unbiased=True)
    assert abs(s_unb / s_pop - np.sqrt(32 / 31)) < 1e-14
    assert abs(s_pop - np.std(a)) < 1e-14 and abs(s_unb - np.std(a, ddof=1)) < 1e-14


def test_chan_merge_of_shards_equals_whole():
    """Global stats over K shards (the multi-rank reading) equal the whole-batch stats."""
    rng = np.random.default_rng(4)
    shards = [rng.normal(i, 1 + i, 100 + 13 * i) for i in range(4)]
    n, mean, m2 = 0, 0.0, 0.0
    for s in shards:                     # Chan et al. pairwise merge, rank order
        nb = s.size
        mb, m2b = oracle.moments(s)
        delta = mb - mean
        tot = n + nb
        mean = mean + delta * nb / tot
        m2 = m2 + m2b + delta * delta * n * nb / tot
        n = tot
    mu, m2w = oracle.moments(np.concatenate(shards))
    assert abs(mean - mu) < 1e-13 and abs(m2 - m2w) < 1e-10 * m2w
