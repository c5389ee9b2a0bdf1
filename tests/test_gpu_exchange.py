"""a2/a6 exchange parity on ONE GPU (driver-verifiable): the production peer-memory kernels
(p2p_allreduce_kernel: two-shot rank-order reduce-scatter + all-gather; p2p_moments_kernel:
rank-order Chan merge) run for K virtual ranks through srl_debug_exchange and are compared
with the oracle's K-shard quantities (SPEC.md S:L505-513 reduce_gradients;
C-A4 global normalisation).

* gradient bucket: rank k's bucket = the oracle's shard-k gradient at scale 1/N_global (C-A14)
  plus its 5 loss sums / N, in fp32.  The exchange must return, on EVERY virtual rank and bit
  for bit, the fp32 sum of those buckets in rank order 0..K-1 (the order DESIGN.md §6 fixes),
  and that sum must equal the oracle's full-batch gradient to fp32 rounding.
* moments: rank k's {n, mean, M2} = oracle_moments of its shard's advantages; every rank's
  merged (mu, sigma) must equal oracle_adv_norm over the union of the shards.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import make_inputs

pytestmark = pytest.mark.gpu


def _shard_buckets(cfg, K, seed=3):
    params, full = make_inputs(cfg, seed=seed)
    shards = [make_inputs(cfg, seed=seed, world=K, rank=k)[1] for k in range(K)]
    advs, rets = [], []
    for sh in shards:
        a, r = oracle.gae(sh["rewards"], sh["values"], sh["dones"], cfg.gamma, cfg.lam)
        advs.append(a.reshape(-1))
        rets.append(r.reshape(-1))
    allA = np.concatenate(advs)
    N = allA.size
    _, mu, sd = oracle.adv_norm(allA)
    buckets, tris = [], []
    for sh, a, r in zip(shards, advs, rets):
        g, sums, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, params, sh["obs"],
                                          sh["actions"], sh["logp_old"], (a - mu) / (sd + 1e-8), r,
                                          cfg.clip_eps, cfg.value_coef, cfg.entropy_coef,
                                          grad_scale=1.0 / N)
        buckets.append(np.concatenate([g, sums / N, [0.0, 0.0, 0.0]]).astype(np.float32))
        m, m2 = oracle.moments(a)
        tris.append([a.size, m, m2])
    o = oracle.ppo_step(cfg, params, [full], apply=False)
    return buckets, np.array(tris), (mu, sd), o


@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_exchange_equals_rank_order_sum_of_oracle_shards(K, op):
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("gfootball").with_(B=16)
    buckets, tris, (mu, sd), o = _shard_buckets(cfg, K)
    count = buckets[0].size                      # P + 8: ragged (not a multiple of 4)
    ld = (count + 63) // 64 * 64
    x = np.zeros((K, ld), np.float32)
    for k in range(K):
        x[k, :count] = buckets[k]
    scale = np.float32(1.0 / K) if op == "mean" else np.float32(1.0)
    out, ms = P.debug_exchange(torch.from_numpy(x).cuda(), scale=float(scale),
                               tri=torch.from_numpy(tris).cuda())
    out = out.cpu().numpy()[:, :count]
    ref = buckets[0].copy()
    for k in range(1, K):
        ref = ref + buckets[k]                   # fp32, rank order 0..K-1
    ref = ref * scale
    for k in range(K):                           # bit-identical on every rank, = rank-order sum
        assert np.array_equal(out[k], ref), (k, np.flatnonzero(out[k] != ref)[:8])
    # ... which is the oracle's full-batch gradient (C-5) up to fp32 rounding of K terms
    G = out[0, :cfg.n_params].astype(np.float64) / float(scale)
    assert np.linalg.norm(G - o["grad"]) <= 1e-6 * np.linalg.norm(o["grad"])
    assert np.allclose(out[0, cfg.n_params:cfg.n_params + 5] / scale, o["sums"] / o["N"], rtol=1e-5, atol=1e-7)
    ms = ms.cpu().numpy()
    for k in range(K):
        assert np.array_equal(ms[k], ms[0])
    assert abs(ms[0, 0] - mu) <= 1e-12 * sd and abs(ms[0, 1] - sd) <= 1e-12 * sd
    assert abs(ms[0, 0] - o["mean"]) <= 1e-12 * sd and abs(ms[0, 1] - o["std"]) <= 1e-12 * sd


@pytest.mark.parametrize("K,count", [(1, 5), (3, 1), (5, 37), (8, 4 * 148 * 1024 + 3), (8, 3_713_070)])
def test_exchange_sizes_and_unbiased(K, count):
    """Ragged / tiny / large (HnS-sized bucket P+8 = 3,713,070) buckets and K that do not
    divide the bucket: every entry is the rank-order fp32 sum; N-1 sigma (C-A4 flag)."""
    import paper_2306_16688_b200 as P
    rng = np.random.default_rng(K * 1000 + count % 997)
    ld = (count + 3) // 4 * 4
    x = rng.normal(size=(K, ld)).astype(np.float32)
    ref = x[0, :count].copy()
    for k in range(1, K):
        ref = ref + x[k, :count]
    n = rng.integers(1, 1000, K).astype(np.float64)
    data = [rng.normal(3.0, 2.0, int(m)) for m in n]
    tris = np.array([[d.size, *oracle.moments(d)] for d in data])
    out, ms = P.debug_exchange(torch.from_numpy(x).cuda(), tri=torch.from_numpy(tris).cuda(),
                               unbiased=True)
    out = out.cpu().numpy()
    for k in range(K):
        assert np.array_equal(out[k, :count], ref)
    allx = np.concatenate(data)
    _, mu, sd = oracle.adv_norm(allx, unbiased=True)
    ms = ms.cpu().numpy()
    assert abs(ms[0, 0] - mu) <= 1e-12 * sd and abs(ms[0, 1] - sd) <= 1e-12 * sd


def test_exchange_rejects_bad_args():
    import paper_2306_16688_b200 as P
    L = P.lib()
    assert L.srl_debug_exchange(9, 4, 4, None, None, 1.0, None, None, 0, None) == P.srl.SRL_EINVAL
    x = torch.zeros((2, 6), device="cuda")
    assert L.srl_debug_exchange(2, 6, 6, x.data_ptr(), x.data_ptr(), 1.0, None, None, 0, None) == P.srl.SRL_EINVAL


def test_allreduce_grads_world1_identity():
    """srl_allreduce_grads with data on a one-rank context: sum and mean are the identity."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("tiny")
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=32)
    buf = torch.randn(1000, device="cuda")
    ref = buf.clone()
    ctx.allreduce_grads(buf, op=0)
    ctx.allreduce_grads(buf, op=1)
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)
    assert ctx.comm_path == "none"
