"""Full-size (Atari-shaped) gradient error vs the oracle under: tanh MUFU / accurate, and the
bench recipe / kink-free recipe.  Oracle work runs over column shards in a process pool."""
import multiprocessing as mp
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import oracle, synth
from ppo_harness import grad_errors, kink_free_xi

cfg = synth.get_config("atari")
W = 16

def lp_shard(r):
    b = synth.make_batch(cfg, seed=0, world=W, rank=r)
    return r, oracle.log_pi(cfg, PARAMS, b["obs"], b["actions"]), b["xi"]

def grad_shard(args):
    r, lo, mean, std = args
    b = synth.make_batch(cfg, seed=0, world=W, rank=r)
    adv, ret = oracle.gae(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam)
    g, sums, _ = oracle.loss_and_grad(cfg.obs_dim, cfg.hidden, cfg.heads, PARAMS, b["obs"], b["actions"], lo,
                                      (adv.reshape(-1) - mean) / (std + 1e-8), ret.reshape(-1), grad_scale=1.0 / cfg.N)
    return r, g

PARAMS = synth.make_params(cfg, 0)

def shard_to_full(parts, Bk):
    # parts: per-rank arrays in local sample order (t*Bk + b) -> full order (t*B + c0 + b)
    T = cfg.T
    return np.concatenate([p.reshape(T, Bk) for p in parts], axis=1).reshape(-1)

def main():
    import paper_2306_16688_b200 as P
    full = synth.make_batch(cfg, seed=0)
    ra, _ = oracle.gae(full["rewards"], full["values"], full["dones"], cfg.gamma, cfg.lam)
    _, mean, std = oracle.adv_norm(ra)
    pool = mp.get_context("fork").Pool(os.cpu_count())
    lps = sorted(pool.map(lp_shard, range(W)), key=lambda x: x[0])
    Bk = cfg.B // W
    lp_full = shard_to_full([x[1] for x in lps], Bk)
    for recipe in ("bench", "kinkfree"):
        if recipe == "bench":
            lo_full = synth.logp_old_uniform_policy(cfg, full["xi"]).astype(np.float64)
        else:
            xi = lp_full - synth.logp_old_uniform_policy(cfg, full["xi"]).astype(np.float64)
            lo_full = lp_full - kink_free_xi(cfg, xi)
        lo32 = lo_full.astype(np.float32)
        lo_sh = [lo32.reshape(cfg.T, cfg.B)[:, r * Bk:(r + 1) * Bk].reshape(-1).astype(np.float64) for r in range(W)]
        gs = sorted(pool.map(grad_shard, [(r, lo_sh[r], mean, std) for r in range(W)]), key=lambda x: x[0])
        gref = sum(g for _, g in gs)
        for tanh in ("mufu", "accurate"):
            os.environ["SRL_TANH"] = tanh
            # fresh process state for the env switch: the library reads it once -> use subprocess
            import subprocess, json, tempfile
            np.save("/tmp/lo.npy", lo32); np.save("/tmp/gref.npy", gref)
            out = subprocess.run([sys.executable, __file__, "gpu"], capture_output=True, text=True, env=dict(os.environ))
            print(recipe, tanh, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:], flush=True)

def gpu():
    import paper_2306_16688_b200 as P
    full = synth.make_batch(cfg, seed=0)
    full["logp_old"] = np.load("/tmp/lo.npy")
    gref = np.load("/tmp/gref.npy")
    d = {k: torch.from_numpy(np.ascontiguousarray(full[k])).cuda() for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}
    adv, ret, st = P.gae(d["rewards"], d["values"], d["dones"], cfg.gamma, cfg.lam)
    ms = P.adv_norm(adv.view(-1), local_stats=st)
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=full["n"])
    ctx.load_params(torch.from_numpy(PARAMS).cuda())
    ctx.step(full["n"], d["obs"], d["actions"], d["logp_old"], adv.view(-1), ret.view(-1), ms, apply=False)
    G = ctx.grads().cpu().numpy().astype(np.float64)[:cfg.n_params]
    e = grad_errors(cfg, G, gref)
    print({k: (round(v[0], 6), round(v[1], 6)) for k, v in e.items()})

if __name__ == "__main__":
    gpu() if len(sys.argv) > 1 else main()
