"""The N>1 path's host-side logic on CPU with world_size 2 over gloo (no GPU needed):
unique-id broadcast, disjoint column shards, the rank-order merge of normalisation moments
and the pre-scaled gradient sum -- checked against the oracle on the full batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _chan(parts):
    n, mean, m2 = 0.0, 0.0, 0.0
    for nb, mb, qb in parts:              # rank order, same fold the CUDA merge kernel uses
        if nb == 0:
            continue
        tot = n + nb
        d = mb - mean
        mean = mean + d * (nb / tot)
        m2 = m2 + qb + d * d * (n * nb / tot)
        n = tot
    return n, mean, m2


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2306_16688_b200.dist import broadcast_unique_id
    try:
        # 1. unique-id broadcast
        uid = broadcast_unique_id(make_id=lambda: bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)))
        # 2. this rank's shard of a gfootball-shaped batch (weak layout: columns split by rank)
        cfg = synth.get_config("gfootball").with_(B=8)
        params = synth.make_params(cfg, 0)
        sh = synth.make_batch(cfg, seed=4, world=world, rank=rank)
        sh["logp_old"] = (oracle.log_pi(cfg, params, sh["obs"], sh["actions"]) - sh["xi"]).astype(np.float32)
        adv, ret = oracle.gae(sh["rewards"], sh["values"], sh["dones"], cfg.gamma, cfg.lam)
        adv, ret = adv.reshape(-1), ret.reshape(-1)
        # 3. moments all-gather, merged in rank order
        mu_l, m2_l = oracle.moments(adv)
        mine = torch.tensor([adv.size, mu_l, m2_l], dtype=torch.float64)
        got = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(got, mine)
        n, mean, m2 = _chan([tuple(g.tolist()) for g in got])
        std = np.sqrt(m2 / n)
        # 4. local gradient pre-scaled by 1/N_global, summed over ranks
        grad, sums, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, params, sh["obs"],
                                             sh["actions"], sh["logp_old"], (adv - mean) / (std + 1e-8),
                                             ret, grad_scale=1.0 / n)
        g = torch.from_numpy(np.concatenate([grad, sums / n]))
        dist.all_reduce(g)
        q.put((rank, uid, sh["c0"], sh["c1"], float(n), mean, std, g.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo_match_full_batch():
    import oracle
    import synth
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # same id on both ranks
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128
    # disjoint, contiguous, covering column blocks
    cfg = synth.get_config("gfootball").with_(B=8)
    assert res[0][2] == 0 and res[0][3] == res[1][2] and res[1][3] == cfg.B
    # global moments and reduced gradient equal the oracle's full batch (C-5)
    params = synth.make_params(cfg, 0)
    full = synth.make_batch(cfg, seed=4)
    full["logp_old"] = (oracle.log_pi(cfg, params, full["obs"], full["actions"]) - full["xi"]).astype(np.float32)
    o = oracle.ppo_step(cfg, params, [full], apply=False)
    for r in res:
        assert r[4] == o["N"]
        assert abs(r[5] - o["mean"]) < 1e-12 * max(1, abs(o["mean"]))
        assert abs(r[6] - o["std"]) < 1e-12 * o["std"]
        g = r[7]
        P = cfg.n_params
        assert np.linalg.norm(g[:P] - o["grad"]) <= 1e-12 * np.linalg.norm(o["grad"])
        np.testing.assert_allclose(g[P:], o["sums"] / o["N"], rtol=1e-12, atol=1e-15)
    # both ranks hold bit-identical reduced results
    assert np.array_equal(res[0][7], res[1][7])
