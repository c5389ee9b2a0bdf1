"""a1 GAE kernel parity vs the oracle (C-T1 mixed metric; C-B1..C-B5 bit-exact cases)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(r, v, d, g, lam, ld=None):
    import paper_2306_16688_b200 as P
    adv, ret, st = P.gae(_dev(r), _dev(v), _dev(d), g, lam, ld=ld)
    torch.cuda.synchronize()
    return adv.cpu().numpy(), ret.cpu().numpy(), st.cpu().numpy()


def _mixed_ok(a, ref, tol=1e-5):
    rms = np.sqrt(np.mean(ref ** 2))
    return np.all(np.abs(a - ref) <= tol * (np.abs(ref) + rms))


@pytest.mark.parametrize("name", ["tiny", "atari", "gfootball", "smac", "hns"])
@pytest.mark.parametrize("stress", [False, True])
def test_gae_configs_reduced_B(name, stress):
    cfg = synth.get_config(name)
    B = min(cfg.B, 96 * cfg.agents if cfg.agents > 1 else 96)
    cfg = cfg.with_(B=B)
    b = synth.make_batch(cfg, seed=3, stress=stress, with_obs=False)
    adv, ret, st = _run(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam)
    ra, rr = oracle.gae(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam)
    assert _mixed_ok(adv, ra) and _mixed_ok(ret, rr)
    mu, m2 = oracle.moments(ra)
    assert st[0] == ra.size
    assert abs(st[1] - mu) <= 1e-5 * (abs(mu) + np.sqrt(m2 / ra.size))
    assert abs(st[2] - m2) <= 1e-4 * m2


@pytest.mark.parametrize("T,B", [(1, 1), (7, 33), (128, 1024), (257, 65), (400, 100), (1500, 40)])
def test_gae_integer_bit_exact(T, B):
    """C-B1: gamma = lambda = 1, small integers, random dones: all values exact in fp32."""
    rng = np.random.default_rng(T * 1000 + B)
    r = rng.integers(-3, 4, (T, B)).astype(np.float32)
    v = rng.integers(-5, 6, (T + 1, B)).astype(np.float32)
    d = (rng.random((T, B)) < 0.05).astype(np.uint8)
    adv, ret, _ = _run(r, v, d, 1.0, 1.0)
    ra, rr = oracle.gae(r, v, d, 1.0, 1.0)
    assert np.array_equal(adv, ra.astype(np.float32)) and np.array_equal(ret, rr.astype(np.float32))


def test_gae_lambda0_and_all_done_exact():
    """C-B2 (lambda = 0, gamma = 0.5 -> A = delta) and C-B3 (all done -> A = r - v)."""
    rng = np.random.default_rng(5)
    T, B = 64, 77
    r = rng.integers(-3, 4, (T, B)).astype(np.float32)
    v = rng.integers(-5, 6, (T + 1, B)).astype(np.float32)
    d = (rng.random((T, B)) < 0.1).astype(np.uint8)
    adv, _, _ = _run(r, v, d, 0.5, 0.0)
    ra, _ = oracle.gae(r, v, d, 0.5, 0.0)
    assert np.array_equal(adv, ra.astype(np.float32))
    adv, _, _ = _run(r, v, np.ones_like(d), 0.99, 0.95)
    assert np.array_equal(adv, r - v[:-1])


def test_gae_index_signature_and_ld_padding():
    """C-B4: r[t][b] = 1000 t + b, v = 0, gamma = 0 -> A = r exactly; padded row stride."""
    T, B, ld = 400, 300, 320
    r = np.zeros((T, ld), np.float32)
    r[:, :B] = (1000 * np.arange(T)[:, None] + np.arange(B)[None, :]).astype(np.float32)
    r[:, B:] = np.nan          # padding must never be read into valid columns
    v = np.zeros((T + 1, ld), np.float32)
    d = np.zeros((T, ld), np.uint8)
    adv, _, _ = _run(r, v, d, 0.0, 0.95, ld=B)
    assert np.array_equal(adv[:, :B], r[:, :B])


def test_gae_shards_concatenate_bit_exact():
    """C-B5: K shards' outputs are the column blocks of the K=1 output, bit for bit."""
    cfg = synth.get_config("smac").with_(B=80 * 10 // 10 * 10)
    full = synth.make_batch(cfg, seed=1, with_obs=False)
    a1, _, _ = _run(full["rewards"], full["values"], full["dones"], cfg.gamma, cfg.lam)
    parts = []
    for k in range(4):
        sh = synth.make_batch(cfg, seed=1, world=4, rank=k, with_obs=False)
        ak, _, _ = _run(sh["rewards"], sh["values"], sh["dones"], cfg.gamma, cfg.lam)
        parts.append(ak)
    assert np.array_equal(np.concatenate(parts, 1), a1)


def test_gae_full_size_smac_sampled_columns():
    """Full SMAC-shaped scan [400 x 20480]: sampled columns vs the oracle."""
    cfg = synth.get_config("smac")
    b = synth.make_batch(cfg, seed=2, with_obs=False)
    adv, ret, st = _run(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam)
    cols = np.random.default_rng(0).choice(cfg.B, 64, replace=False)
    ra, rr = oracle.gae(b["rewards"][:, cols], b["values"][:, cols], b["dones"][:, cols],
                        cfg.gamma, cfg.lam)
    assert _mixed_ok(adv[:, cols], ra) and _mixed_ok(ret[:, cols], rr)
    assert st[0] == cfg.N
