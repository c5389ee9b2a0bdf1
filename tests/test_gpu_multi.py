"""a2/a6 over real NCCL with one process per GPU (needs >= 2 GPUs; skipped otherwise):
K ranks' train steps on disjoint column shards give bit-identical parameters on every rank,
a global normalisation identical to the full batch, and the full-batch oracle gradient."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, p2p="1", steps=1):
    import sys
    # "1u": the peer path with the exchange as its own launch between two update launches
    # (SRL_XFUSED=0) instead of inside the update launch
    os.environ["SRL_XFUSED"] = "0" if p2p == "1u" else "1"
    p2p = "1" if p2p == "1u" else p2p
    os.environ["SRL_P2P_AR"] = p2p
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import synth
        import paper_2306_16688_b200 as P
        from paper_2306_16688_b200.dist import broadcast_unique_id
        from ppo_harness import make_inputs, to_dev
        cfg = synth.get_config("gfootball").with_(B=16)
        params, sh = make_inputs(cfg, seed=3, world=world, rank=rank)
        uid = broadcast_unique_id(device=torch.device("cuda", rank))
        ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=sh["n"], rank=rank, world=world,
                           nccl_id=uid, device=rank)
        ctx.load_params(torch.from_numpy(params).cuda())
        d = to_dev(sh)
        st = P.decode_stats(ctx.train_step(cfg.N, d["rewards"], d["values"], d["dones"], d["obs"],
                                           d["actions"], d["logp_old"]))
        g1 = ctx.grads().cpu().numpy()
        for _ in range(steps - 1):       # both buffer parities of the peer path, epochs advance
            ctx.train_step(cfg.N, d["rewards"], d["values"], d["dones"], d["obs"], d["actions"],
                           d["logp_old"])
        torch.cuda.synchronize()
        q.put((rank, st, ctx.params().cpu().numpy(), g1, ctx.comm_path))
        ctx.close()
    finally:
        dist.destroy_process_group()


def _run(world, p2p="1", steps=1):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, p2p, steps)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_nccl_ranks_match_full_batch(world, p2p):
    """p2p = 1: the gradient bucket is reduced by the NVLink peer-memory kernel (default);
    p2p = 0: by NCCL.  Both must give the full-batch result on every rank."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import synth
    from ppo_harness import grad_errors, make_inputs
    res = _run(world, p2p)
    assert res[0][4] == ("nvlink-p2p" if p2p == "1" else "nccl")
    cfg = synth.get_config("gfootball").with_(B=16)
    params, full = make_inputs(cfg, seed=3)
    o = oracle.ppo_step(cfg, params, [full], apply=False)
    for r in res[1:]:                                     # S:L522 parameters bit-identical
        assert np.array_equal(r[2], res[0][2]) and np.array_equal(r[3], res[0][3])
    st = res[0][1]
    assert st["n_global"] == cfg.N and st["step"] == 1
    assert abs(st["adv_mean"] - o["mean"]) <= 1e-6 * o["std"] and abs(st["adv_std"] - o["std"]) <= 1e-6 * o["std"]
    G = res[0][3][:cfg.n_params].astype(np.float64)
    errs = grad_errors(cfg, G, o["grad"])
    assert all(v[0] <= 2e-3 and v[1] <= 2e-3 for v in errs.values()), errs


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_allreduce_equals_nccl_over_steps(world):
    """Three steps (both exposed-buffer parities): the peer-memory reduction (rank-order sum)
    and NCCL's agree to fp32 rounding on the first gradient and on the final parameters."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    a = _run(world, "1", steps=3)
    b = _run(world, "0", steps=3)
    assert a[0][4] == "nvlink-p2p" and b[0][4] == "nccl"
    for r in a[1:]:
        assert np.array_equal(r[2], a[0][2])
    ga, gb = a[0][3].astype(np.float64), b[0][3].astype(np.float64)
    assert np.linalg.norm(ga - gb) <= 1e-6 * np.linalg.norm(gb)
    # Adam normalises each entry: a gradient entry within rounding of 0 may take either sign,
    # moving that parameter by up to 2 lr per step; everything else agrees to rounding
    d = np.abs(a[0][2].astype(np.float64) - b[0][2].astype(np.float64))
    assert d.max() <= 2 * 3e-4 * 3 + 1e-6 and np.mean(d > 1e-5) <= 1e-3
    assert a[0][1]["step"] == 1 and b[0][1]["step"] == 1


@pytest.mark.parametrize("world", [2, 4])
def test_fused_exchange_equals_three_launches(world):
    """The a6 exchange inside the update launch (default) and as its own launch between the
    finalise and Adam launches (SRL_XFUSED=0) do the same arithmetic (rank-order sum per entry,
    whatever the sub-block partition): bit-identical gradients and parameters after 3 steps."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    a = _run(world, "1", steps=3)
    b = _run(world, "1u", steps=3)
    assert a[0][4] == "nvlink-p2p" and b[0][4] == "nvlink-p2p"
    for ra, rb in zip(a, b):
        assert np.array_equal(ra[3], rb[3]) and np.array_equal(ra[2], rb[2])
        assert ra[1]["step"] == rb[1]["step"] == 1 and ra[1]["comm_error"] == 0


def _api_worker(rank, world, port, q, p2p):
    """srl_allreduce_grads (op 0 / 1, a bucket-sized buffer on the peer path and an oversized
    one through NCCL) and srl_adv_norm(ctx, world > 1) with data on every rank."""
    import sys
    os.environ["SRL_P2P_AR"] = p2p
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import synth
        import paper_2306_16688_b200 as P
        from paper_2306_16688_b200.dist import broadcast_unique_id
        cfg = synth.get_config("gfootball").with_(B=16)
        uid = broadcast_unique_id(device=torch.device("cuda", rank))
        ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=cfg.T * cfg.B // world,
                           rank=rank, world=world, nccl_id=uid, device=rank)
        res = {"path": ctx.comm_path}
        for name, count in (("small", ctx.P + 8), ("big", 3 * ctx.P + 5)):
            for op in (0, 1):
                g = torch.Generator().manual_seed(1000 * op + count)
                allx = torch.randn((world, count), generator=g)      # every rank's input
                buf = allx[rank].clone().cuda()
                ctx.allreduce_grads(buf, op=op)
                res[(name, op)] = (buf.cpu().numpy(), allx.numpy())
        g = torch.Generator().manual_seed(77)
        alla = torch.randn((world, 5000), generator=g, dtype=torch.float64) * 3 + 1
        adv = alla[rank].float().cuda()
        ms = P.adv_norm(adv, ctx=ctx)
        res["ms"] = (ms.cpu().numpy(), alla.float().double().numpy())
        torch.cuda.synchronize()
        q.put((rank, res))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_allreduce_grads_and_adv_norm_api(world, p2p):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import torch.multiprocessing as mp
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _port()
    procs = [mpc.Process(target=_api_worker, args=(r, world, port, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1]["path"] == ("nvlink-p2p" if p2p == "1" else "nccl")
    for key in [("small", 0), ("small", 1), ("big", 0), ("big", 1)]:
        outs = [r[1][key][0] for r in res]
        allx = res[0][1][key][1]
        ref = allx[0].copy()
        for k in range(1, world):
            ref = ref + allx[k]                       # fp32 rank-order sum
        if key[1] == 1:
            ref = ref * np.float32(1.0 / world)
        for o in outs[1:]:                            # identical on every rank
            assert np.array_equal(o, outs[0])
        if p2p == "1" and key[0] == "small":          # the peer path: rank order, bit-exact
            assert np.array_equal(outs[0], ref)
        else:                                         # NCCL's order: fp32 rounding
            assert np.allclose(outs[0], ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
    ms, alla = res[0][1]["ms"]
    _, mu, sd = oracle.adv_norm(alla.reshape(-1))
    for r in res:
        assert np.array_equal(r[1]["ms"][0], ms)
    assert abs(ms[0] - mu) <= 1e-12 * sd and abs(ms[1] - sd) <= 1e-12 * sd


def _timeout_worker(rank, world, port, q):
    """Rank 1 creates its context but never steps: rank 0's exchange waits time out after
    SRL_COMM_TIMEOUT_S; the step reports comm_error with Adam skipped, the next call fails."""
    import sys
    import time
    os.environ["SRL_COMM_TIMEOUT_S"] = "2"
    os.environ["SRL_P2P_AR"] = "1"
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import synth
        import paper_2306_16688_b200 as P
        from paper_2306_16688_b200.dist import broadcast_unique_id
        from ppo_harness import make_inputs, to_dev
        cfg = synth.get_config("gfootball").with_(B=16)
        params, sh = make_inputs(cfg, seed=3, world=world, rank=rank)
        uid = broadcast_unique_id(device=torch.device("cuda", rank))
        ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=sh["n"], rank=rank, world=world,
                           nccl_id=uid, device=rank)
        ctx.load_params(torch.from_numpy(params).cuda())
        torch.cuda.synchronize()
        out = None
        if rank == 0:
            d = to_dev(sh)
            t0 = time.time()
            st = P.decode_stats(ctx.train_step(cfg.N, d["rewards"], d["values"], d["dones"],
                                               d["obs"], d["actions"], d["logp_old"]))
            waited = time.time() - t0
            try:
                ctx.train_step(cfg.N, d["rewards"], d["values"], d["dones"], d["obs"],
                               d["actions"], d["logp_old"])
                err = ""
            except P.SrlError as e:
                err = str(e)
            out = (st["comm_error"], st["step"], waited, err, ctx.comm_path)
        q.put((rank, out))
        dist.barrier()
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_comm_timeout_reports_enccl():
    """SPEC.md S:L532 ReduceTimeout as SRL_ENCCL: a missing peer makes the
    peer-path waits give up after SRL_COMM_TIMEOUT_S instead of hanging or trapping."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _port()
    procs = [mpc.Process(target=_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    comm_error, step, waited, err, path = res[0][1]
    assert path == "nvlink-p2p"
    assert comm_error == 1 and step == 0                 # Adam skipped
    assert 1.5 <= waited <= 60.0
    assert "status 3" in err                             # SRL_ENCCL on the next call
