"""Pins for oracle C-1 (GAE) against closed forms, brute force and hand values.

DESIGN.md §3.1 / SURVEY.md §8(c) C-1: backward recursion of BASELINE.json north_star.
None of these re-type the recursion: they use SPEC.md's printed example, the
closed forms the north star names (lambda=0 -> one-step TD error; lambda=gamma=1 ->
return minus value; done cuts the recursion) and the direct double sum.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand(T, B, seed, p_done=0.1, integer=False):
    rng = np.random.default_rng(seed)
    if integer:
        r = rng.integers(-3, 4, (T, B)).astype(np.float32)
        v = rng.integers(-5, 6, (T + 1, B)).astype(np.float32)
    else:
        r = rng.normal(size=(T, B)).astype(np.float32)
        v = rng.normal(size=(T + 1, B)).astype(np.float32)
    d = (rng.random((T, B)) < p_done).astype(np.uint8)
    return r, v, d


def test_golden_hand_cases():
    g = json.load(open(os.path.join(GOLD, "gae_hand.json")))
    for c in g["cases"]:
        r = np.array(c["r"], np.float32)[:, None]
        v = np.array(c["v"], np.float32)[:, None]
        d = np.array(c["d"], np.uint8)[:, None]
        adv, ret = oracle.gae(r, v, d, c["gamma"], c["lambda"])
        assert np.array_equal(adv[:, 0], np.array(c["adv"], float)), c["name"]
        assert np.array_equal(ret[:, 0], np.array(c["ret"], float)), c["name"]


def test_lambda_zero_is_one_step_td():
    r, v, d = _rand(40, 7, 1)
    adv, _ = oracle.gae(r, v, d, 0.97, 0.0)
    r64, v64, m = r.astype(float), v.astype(float), 1.0 - d
    td = r64 + 0.97 * v64[1:] * m - v64[:-1]
    np.testing.assert_allclose(adv, td, rtol=0, atol=1e-14)


def test_gamma_lambda_one_no_done_is_return_minus_value():
    r, v, _ = _rand(30, 5, 2)
    d = np.zeros_like(r, dtype=np.uint8)
    adv, ret = oracle.gae(r, v, d, 1.0, 1.0)
    r64, v64 = r.astype(float), v.astype(float)
    # telescoping: A_t = sum_{k>=t} r_k + v_T - v_t
    tail = np.cumsum(r64[::-1], axis=0)[::-1]
    np.testing.assert_allclose(adv, tail + v64[-1] - v64[:-1], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ret, tail + v64[-1], rtol=0, atol=1e-12)


def test_all_done_is_reward_minus_value():
    r, v, _ = _rand(12, 6, 3)
    d = np.ones_like(r, dtype=np.uint8)
    adv, _ = oracle.gae(r, v, d, 0.99, 0.95)
    np.testing.assert_array_equal(adv, r.astype(float) - v[:-1].astype(float))


def _bruteforce(r, v, d, g, lam):
    """A_t = sum_k (g lam)^k (prod_{j=t}^{t+k-1} m_j) delta_{t+k}  (S:L601 double sum)."""
    T, B = r.shape
    r, v, m = r.astype(float), v.astype(float), 1.0 - d.astype(float)
    out = np.zeros((T, B))
    for b in range(B):
        for t in range(T):
            s = 0.0
            for k in range(T - t):
                coef = (g * lam) ** k
                for j in range(t, t + k):
                    coef *= m[j, b]
                tk = t + k
                delta = r[tk, b] + g * v[tk + 1, b] * m[tk, b] - v[tk, b]
                s += coef * delta
            out[t, b] = s
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bruteforce_double_sum(seed):
    r, v, d = _rand(50, 3, 10 + seed, p_done=0.08)
    adv, _ = oracle.gae(r, v, d, 0.99, 0.95)
    bf = _bruteforce(r, v, d, 0.99, 0.95)
    scale = np.abs(bf).max()
    assert np.abs(adv - bf).max() <= 1e-12 * max(scale, 1.0)


def test_done_cuts_future():
    r, v, d = _rand(20, 4, 4, p_done=0.0)
    d[9, :] = 1
    a1, _ = oracle.gae(r, v, d, 0.9, 0.8)
    r2, v2 = r.copy(), v.copy()
    r2[10:] += 5.0
    v2[10:] -= 3.0          # v_{10..T}: v_10 is v_{t+1} of the done step -> masked
    a2, _ = oracle.gae(r2, v2, d, 0.9, 0.8)
    np.testing.assert_array_equal(a1[:10], a2[:10])
    # at the done step itself: A_t = r_t - v_t
    np.testing.assert_array_equal(a1[9], r[9].astype(float) - v[9].astype(float))


def test_linearity_integer_exact():
    r1, v1, d = _rand(25, 5, 5, integer=True)
    r2, v2, _ = _rand(25, 5, 6, integer=True)
    a1, _ = oracle.gae(r1, v1, d, 0.5, 0.5)
    a2, _ = oracle.gae(r2, v2, d, 0.5, 0.5)
    a12, _ = oracle.gae(r1 + r2, v1 + v2, d, 0.5, 0.5)
    np.testing.assert_allclose(a12, a1 + a2, rtol=0, atol=1e-12)


def test_integer_gamma_lambda_one_exact_integers():
    """C-B1 fixture: gamma=lambda=1 and small integers keep every value an exact integer."""
    r, v, d = _rand(64, 9, 7, integer=True, p_done=0.2)
    adv, ret = oracle.gae(r, v, d, 1.0, 1.0)
    assert np.array_equal(adv, np.round(adv)) and np.abs(adv).max() < 2 ** 24
