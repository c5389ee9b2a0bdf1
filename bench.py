#!/usr/bin/env python3
"""Benchmark: PPO trainer samples/sec for the whole hot path (GAE -> normalisation ->
forward -> loss -> backward -> allreduce -> Adam) on synthetic Atari-shaped batches.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config atari] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Scaling is weak: every rank trains its own full config-shaped shard (T x B columns); the
ranks' shards are disjoint column blocks of one global batch, normalised globally and
reduced by one allreduce of the gradient bucket per step (the library's NVLink peer-memory
kernel by default, NCCL with SRL_P2P_AR=0).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "PPO trainer samples/sec (GAE+update, device-timed) at 1/2/4/8 B200"
_OUT_FD = None


def emit(obj):
    line = (json.dumps(obj) + "\n").encode()
    if _OUT_FD is not None:
        os.write(_OUT_FD, line)
    else:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="atari")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps (capped at 100)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    # NEXT-3 PPO variants (defaults = the BASELINE workload: one update per batch, no clipping)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--minibatches", type=int, default=1)
    ap.add_argument("--value-clip", type=float, default=0.0)
    ap.add_argument("--max-grad-norm", type=float, default=0.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_ids):
        self.ids = ",".join(str(i) for i in gpu_ids)
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", self.ids, "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self, t0, t1):
        win = [s for t, s in self.samples if t0 - 0.06 <= t <= t1 + 0.06]
        note = "timed-region samples"
        if not win:
            win = [s for _, s in self.samples]
            note = "no sample inside the timed region; samples from the whole run"
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": "nvidia-smi unavailable"}
        sm = [float(s[1]) for s in win if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in win if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in win for k in range(4) if s[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(win), "note": note}


# ------------------------------------------------------------------ CPU oracle
def time_oracle(cfg, budget_s, params=None):
    """The oracle (as it stands, 1 thread) on a bounded sample of the workload: T x B' columns
    with B' chosen so the run takes about budget_s.  Returns (samples/s, n, B', seconds)."""
    import oracle
    import synth
    if params is None:
        params = synth.make_params(cfg, 0)

    def run(Bp):
        c = cfg.with_(B=Bp * cfg.agents)
        b = synth.make_batch(c, seed=0)
        b["logp_old"] = synth.logp_old_uniform_policy(c, b["xi"])
        t = time.perf_counter()
        oracle.ppo_step(c, params, [b], apply=True)
        return time.perf_counter() - t, b["n"]

    t1, n1 = run(1)
    Bp = int(max(1, min(cfg.B // cfg.agents, round(budget_s / max(t1, 1e-6)))))
    if Bp == 1:
        return n1 / t1, n1, 1, t1
    t, n = run(Bp)
    return n / t, n, Bp, t


def reference_arm(args, world, rank):
    """--impl reference: the oracle as it stands, on this box's host cores, same metric/unit."""
    import synth
    cfg = synth.get_config(args.config)
    if rank != 0:
        return
    per_step = max(0.2, 150.0 / max(1, args.steps + args.warmup))
    import oracle
    params = synth.make_params(cfg, 0)
    # calibrate one column, then size the per-step sample
    _, _, _, t1 = time_oracle(cfg, 0.0, params)
    Bp = int(max(1, min(cfg.B // cfg.agents, per_step / max(t1, 1e-6))))
    c = cfg.with_(B=Bp * cfg.agents)
    b = synth.make_batch(c, seed=0)
    b["logp_old"] = synth.logp_old_uniform_policy(c, b["xi"])
    nx = dict(epochs=max(1, args.epochs), minibatches=max(1, args.minibatches),
              value_clip=args.value_clip, max_grad_norm=args.max_grad_norm)
    for _ in range(args.warmup):
        oracle.ppo_step(c, params, [b], apply=True, **nx)
    t0 = time.perf_counter()
    for k in range(args.steps):
        oracle.ppo_step(c, params, [b], apply=True, t=k + 1, **nx)
    dt = time.perf_counter() - t0
    value = b["n"] * args.steps / dt
    sample = (f"{cfg.name}-shaped T={cfg.T}, B'={Bp * cfg.agents} columns ({b['n']} samples) per "
              f"step, full network, GAE+norm+loss/grad+Adam, C double, 1 thread")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": cfg.name, "T": cfg.T, "B_per_step": Bp * cfg.agents, **nx},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# ------------------------------------------------------------------ our arm
def main_ours(args, world, rank, local):
    import torch
    import synth
    import paper_2306_16688_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    cfg = synth.get_config(args.config)
    gcfg = cfg.with_(B=cfg.B * world)          # weak scaling: one config-sized shard per rank
    b = synth.make_batch(gcfg, seed=0, world=world, rank=rank)
    b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
    n = b["n"]
    N = n * world
    params = torch.from_numpy(synth.make_params(cfg, 0)).to(dev)
    keys = ("rewards", "values", "dones", "obs", "actions", "logp_old")
    host = {k: torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys}
    d = {k: host[k].to(dev) for k in keys}
    h2d_bytes = sum(host[k].numel() * host[k].element_size() for k in keys)

    nccl_id = None
    if world > 1:
        from paper_2306_16688_b200.dist import broadcast_unique_id
        nccl_id = broadcast_unique_id(device=dev)
    import dataclasses
    spec = dataclasses.replace(P.NetSpec.from_config(cfg), epochs=args.epochs,
                               minibatches=args.minibatches, value_clip=args.value_clip,
                               max_grad_norm=args.max_grad_norm)
    ctx = P.PPOContext(spec, max_local_n=n, rank=rank, world=world, nccl_id=nccl_id, device=local)
    ctx.load_params(params)
    T, Bk = b["rewards"].shape
    stats = torch.zeros(P.srl.STATS_BYTES, dtype=torch.uint8, device=dev)
    stats_host = torch.zeros(P.srl.STATS_BYTES, dtype=torch.uint8).pin_memory()

    def step(src):
        # one C-ABI call: GAE -> global normalisation -> forward/loss/backward -> allreduce -> Adam
        ctx.train_step(N, src["rewards"], src["values"], src["dones"], src["obs"], src["actions"],
                       src["logp_old"], stats=stats)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step(d)
    barrier()
    sampler = ClockSampler(range(world)) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    # ---------------- timed region: device-resident inputs (working set > L2: see config)
    K = args.steps
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    wall0 = time.monotonic()
    e_start.record()
    h0 = time.perf_counter()
    for _ in range(K):
        step(d)
    host_ms = (time.perf_counter() - h0) * 1e3 / K
    e_end.record()
    barrier()
    wall1 = time.monotonic()
    ms_total = max_over_ranks(e_start.elapsed_time(e_end))
    stats_dev = P.decode_stats(stats)
    # ---------------- profiled region: same steps with an event pair around every launch (the
    # events serialise the launches, so this region is timed separately from `value`)
    Kp = min(K, 100)
    ctx.prof_reset()
    ctx.profile(True)
    p_start, p_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    p_start.record()
    for _ in range(Kp):
        step(d)
    p_end.record()
    barrier()
    ctx.profile(False)
    prof_ms = max_over_ranks(p_start.elapsed_time(p_end)) / Kp
    recs = ctx.prof_records()

    # ---------------- end to end: every step's batch goes host (pinned) -> device inside the timed
    # region through the library's pre-fetch slots (NEXT-1, §4.1): the upload of batch
    # k+1 on the context's copy stream overlaps the step on batch k; stats are copied back
    Ke = args.e2e_steps or min(K, 100)
    hb = [host[k] for k in keys]
    ctx.upload(0, *hb)
    for j in range(2):
        ctx.upload((j + 1) % 2, *hb)
        ctx.train_step_slot(j % 2, N, stats=stats)
        stats_host.copy_(stats, non_blocking=True)
    ctx.train_step_slot(0, N, stats=stats)          # drain the primed slot
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record()
    ctx.upload(0, *hb)
    for j in range(Ke):
        if j + 1 < Ke:
            ctx.upload((j + 1) % 2, *hb)
        ctx.train_step_slot(j % 2, N, stats=stats)
        stats_host.copy_(stats, non_blocking=True)
    x1.record()
    barrier()
    e2e_ms = max_over_ranks(x0.elapsed_time(x1))
    # ---------------- NEXT-2: policy-worker batched inference on the same batch of observations
    # (forward + counter-RNG sampling epilogue), device-timed like `value`
    Ki = min(K, 100)
    inf_out = (torch.empty((n, len(cfg.heads)), dtype=torch.int32, device=dev),
               torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.float32, device=dev))
    for j in range(3):
        ctx.rollout(d["obs"], seed=j, actions=inf_out[0], logp=inf_out[1], value=inf_out[2])
    barrier()
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record()
    for j in range(Ki):
        ctx.rollout(d["obs"], seed=j, actions=inf_out[0], logp=inf_out[1], value=inf_out[2])
    i1.record()
    barrier()
    inf_ms = max_over_ranks(i0.elapsed_time(i1)) / Ki
    if sampler:
        time.sleep(0.1)
        sampler.stop()

    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---------------- per-kernel table and the dominant kernel's roofline
    import math
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tf_sus = float(peaks.get("bf16_tflops_sustained", 1400.0))
    peak_src = "measured" if peaks else "fallback"
    agg = {}
    for name, t, fl, by in recs:
        a = agg.setdefault(name, [0.0, 0, 0.0, 0.0])
        a[0] += t; a[1] += 1; a[2] += fl; a[3] += by
    step_ms = ms_total / K
    kernels = []
    for name, (t, cnt, fl, by) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        avg = t / max(cnt, 1)
        row = {"name": name, "ms_per_step": t / Kp, "share": (t / Kp) / prof_ms, "launches_per_step": cnt / Kp}
        if fl > 0:
            row.update(tflops=fl / cnt / (avg * 1e-3) / 1e12, frac_tensor=fl / cnt / (avg * 1e-3) / 1e12 / tf_sus)
        if by > 0:
            row.update(gbs=by / cnt / (avg * 1e-3) / 1e9, frac_hbm=by / cnt / (avg * 1e-3) / 1e9 / hbm)
        kernels.append(row)
    # dominant kernel by time; its roof is the one its arithmetic intensity (algorithmic FLOP per
    # algorithmic HBM byte) puts it under: tensor above the ridge (peak FLOP/s / peak B/s), else HBM
    dname, (dt, dcnt, dfl, dby) = max(((k, v) for k, v in agg.items() if k != "allreduce"),
                                      key=lambda kv: kv[1][0])   # NCCL's kernel is not ours
    davg_s = dt / dcnt * 1e-3
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(args.config, {}).get(dname)
    except Exception:
        pass
    ridge = tf_sus * 1e12 / (hbm * 1e9)
    ai = dfl / dby if dby > 0 else float("inf")
    if dfl > 0 and ai >= ridge:
        achieved = dfl / dcnt / davg_s / 1e12
        roofline = {"bound": "tensor", "kernel": dname, "achieved": achieved, "peak": tf_sus,
                    "unit": "TFLOP/s", "frac": achieved / tf_sus, "traffic": traffic,
                    "peak_source": f"{peak_src} bf16_tflops_sustained (fp16 dense = bf16 dense, nominal ratio 1)"}
    else:
        achieved = dby / dcnt / davg_s / 1e9
        roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm,
                    "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                    "peak_source": f"{peak_src} hbm_gbs (copy)"}
    roofline.update(flops_per_launch=dfl / dcnt, bytes_per_launch=dby / dcnt,
                    intensity_flop_per_byte=ai, ridge_flop_per_byte=ridge,
                    ms_per_launch=davg_s * 1e3)
    # our kernels per step (srl_ppo_train_step): gae_kernel (merges the moments itself),
    # + moments merge when world > 1, the 3L+2 GEMMs, finalize_w + finalize_b + extras, adam,
    # stats (NCCL's kernels are not counted)
    L = len(cfg.hidden)
    # per update; epochs x minibatches updates per step (NEXT-3), + grad_norm when clipping
    p2p = ctx.comm_path == "nvlink-p2p"      # the allreduce is then one of our kernels
    per_update = ((L + 1 + (L + 1) + L) + 3 + 1 + 1 + (1 if args.max_grad_norm > 0 else 0)
                  + (1 if p2p else 0))
    updates = max(1, args.epochs) * max(1, args.minibatches)
    per_step = 1 + (1 if world > 1 else 0) + per_update * updates
    cpu = None
    if not args.no_cpu_baseline:
        v, cn, Bp, secs = time_oracle(cfg, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{cfg.name}-shaped T={cfg.T}, B'={Bp * cfg.agents} columns ({cn} samples; "
                         f"{secs:.1f} s), full network, GAE+norm+loss/grad+Adam, C double, 1 thread"}
    clocks = sampler.summary(wall0, wall1) if sampler else None
    out = {
        "metric": METRIC, "value": N * K / (ms_total * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": max(3, args.warmup), "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic",
        "config": {"workload": cfg.name, "T": cfg.T, "B_per_rank": cfg.B, "obs_dim": cfg.obs_dim,
                   "hidden": list(cfg.hidden), "heads": list(cfg.heads), "samples_per_step": N,
                   "frames_per_step": N * cfg.frame_skip, "parallelism": f"dp{world}",
                   "grad_allreduce": ctx.comm_path,
                   "epochs": max(1, args.epochs), "minibatches": max(1, args.minibatches),
                   "value_clip": args.value_clip, "max_grad_norm": args.max_grad_norm,
                   "l2": "no flush: per-step working set > L2 (obs %.0f MB + activations %.0f MB + "
                         "dZ %.0f MB per rank vs 126 MB L2)" % (
                             n * cfg.ld_obs * 2 / 1e6, n * sum(cfg.hidden) * 2 / 1e6,
                             n * max(cfg.hidden) * 4 / 1e6)},
        "frames_per_s": N * cfg.frame_skip * K / (ms_total * 1e-3),
        "sample_updates_per_s": N * updates * K / (ms_total * 1e-3),
        "host_submit_ms_per_step": host_ms,
        "profiled_ms_per_step": prof_ms,
        "e2e": {"value": N * Ke / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d_bytes * world,
                "d2h_bytes_per_step": P.srl.STATS_BYTES * world, "steps": Ke},
        "gpu_launches": per_step * K,
        "inference": {"what": "NEXT-2 srl_policy_rollout: forward + sampling epilogue over the "
                              "step's observations (policy-worker batch = the whole batch)",
                      "value": N / (inf_ms * 1e-3), "unit": "samples/s", "ms_per_call": inf_ms,
                      "batch_per_rank": n, "calls": Ki, "gpu_launches_per_call": L + 1},
        "roofline": roofline,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "last_stats": {k: stats_dev[k] for k in ("loss", "policy_loss", "value_loss", "entropy",
                                                 "clip_fraction", "nonfinite", "step")},
    }
    if any(math.isnan(x) for x in (out["value"],)):
        raise SystemExit("nan throughput")
    emit(out)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    # keep stdout for the one JSON line: library / NCCL chatter on fd 1 goes to stderr
    out_fd = os.dup(1)
    os.dup2(2, 1)
    global _OUT_FD
    _OUT_FD = out_fd
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    if args.gpus > 1 and world == 1:
        raise SystemExit("--gpus N > 1: launch with torchrun --nproc-per-node N (one rank per GPU)")
    main_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
