"""a2 advantage normalisation parity vs the oracle (C-T2)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 33, 4096, 1_000_003])
@pytest.mark.parametrize("unbiased", [0, 1])
def test_adv_norm_matches_oracle(n, unbiased):
    import paper_2306_16688_b200 as P
    if n == 1 and unbiased:
        pytest.skip("N-1 undefined")
    rng = np.random.default_rng(n)
    a = (rng.normal(3.0, 2.5, n)).astype(np.float32)
    x = torch.from_numpy(a).cuda()
    ms = P.adv_norm(x, eps=1e-8, unbiased=bool(unbiased), apply=True)
    torch.cuda.synchronize()
    out, mu, sd = oracle.adv_norm(a.astype(np.float64), eps=1e-8, unbiased=unbiased)
    ms = ms.cpu().numpy()
    assert abs(ms[0] - mu) <= 1e-12 * max(1.0, abs(mu))
    assert abs(ms[1] - sd) <= 1e-10 * max(sd, 1e-30) + 1e-300
    got = x.cpu().numpy()
    rms = np.sqrt(np.mean(out ** 2)) if n > 1 else 1.0
    assert np.all(np.abs(got - out) <= 1e-5 * (np.abs(out) + rms))


def test_adv_norm_from_gae_stats():
    import paper_2306_16688_b200 as P
    rng = np.random.default_rng(9)
    T, B = 128, 256
    r = torch.from_numpy(rng.normal(size=(T, B)).astype(np.float32)).cuda()
    v = torch.from_numpy(rng.normal(size=(T + 1, B)).astype(np.float32)).cuda()
    d = torch.from_numpy((rng.random((T, B)) < 0.02).astype(np.uint8)).cuda()
    adv, ret, st = P.gae(r, v, d, 0.99, 0.95)
    ms1 = P.adv_norm(adv, local_stats=st)
    ms2 = P.adv_norm(adv)
    torch.cuda.synchronize()
    ra, _ = oracle.gae(r.cpu().numpy(), v.cpu().numpy(), d.cpu().numpy(), 0.99, 0.95)
    _, mu, sd = oracle.adv_norm(ra)
    for ms in (ms1.cpu().numpy(), ms2.cpu().numpy()):
        assert abs(ms[0] - mu) <= 1e-6 * sd and abs(ms[1] - sd) <= 1e-6 * sd
