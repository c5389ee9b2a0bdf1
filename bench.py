#!/usr/bin/env python3
"""Benchmark: PPO trainer samples/sec for the whole hot path (GAE -> normalisation ->
forward -> loss -> backward -> allreduce -> Adam) on synthetic Atari-shaped batches.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config atari] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Scaling (N > 1): strong by default -- the config's batch is the global batch, split into B/K
column blocks, one per rank (SURVEY C-A16); the other mode (weak: a full config-sized shard per
rank) is measured in the same run under "alt_scaling".  Shards are normalised globally and
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
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    # NEXT-3 PPO variants (defaults = the BASELINE workload: one update per batch, no clipping)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--minibatches", type=int, default=1)
    ap.add_argument("--value-clip", type=float, default=0.0)
    ap.add_argument("--max-grad-norm", type=float, default=0.0)
    ap.add_argument("--separate-critic", action="store_true",
                    help="NEXT-3 R-AC: separate actor and critic trunks (DESIGN.md §3.5)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="default: strong for N > 1 (the config batch split B/K, SURVEY C-A16)")
    ap.add_argument("--no-alt-scaling", action="store_true")
    ap.add_argument("--no-all-configs", action="store_true")
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
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(cfg, Bp):
    import synth
    c = cfg.with_(B=Bp * cfg.agents)
    b = synth.make_batch(c, seed=0)
    b["logp_old"] = synth.logp_old_uniform_policy(c, b["xi"])
    return c, b


def time_oracle(cfg, budget_s, threads=1, params=None, nx=None):
    """The oracle (as it stands; threads > 1 = its all-core block driver) on a bounded sample of
    the workload: T x B' columns, B' sized so one step takes about budget_s.
    Returns (samples/s, n, B', seconds)."""
    import oracle
    import synth
    if params is None:
        params = synth.make_params(cfg, 0)
    nx = nx or {}

    def run(Bp):
        c, b = oracle_sample(cfg, Bp)
        t = time.perf_counter()
        oracle.ppo_step(c, params, [b], apply=True, threads=threads, **nx)
        return time.perf_counter() - t, b["n"]

    Bp0 = max(1, min(cfg.B // cfg.agents, threads))
    t1, n1 = run(Bp0)
    Bp = int(max(1, min(cfg.B // cfg.agents, round(Bp0 * budget_s / max(t1, 1e-6)))))
    if Bp == Bp0:
        return n1 / t1, n1, Bp0, t1
    t, n = run(Bp)
    return n / t, n, Bp, t


def cpu_baselines(cfg, budget_s):
    """1 thread (the parity build) and all host cores (block driver), SURVEY.md §8(d) D-5."""
    cores = host_cores()
    v1, n1, B1, s1 = time_oracle(cfg, budget_s, 1)
    vN, nN, BN, sN = time_oracle(cfg, budget_s, cores)
    model = cpu_model()
    desc = lambda Bp, n, secs, th: (f"{cfg.name}-shaped T={cfg.T}, B'={Bp * cfg.agents} columns ({n} samples; "
                                    f"{secs:.1f} s), full network, GAE+norm+loss/grad+Adam, C double, "
                                    f"{th} thread(s) on {model}")
    return {"value": vN, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": model,
            "sample": desc(BN, nN, sN, cores),
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": desc(B1, n1, s1, 1)}}


def reference_arm(args, world, rank):
    """--impl reference: the oracle as it stands, on this box's host cores (all of them, through
    its block driver), same metric / unit / config as our arm."""
    import synth
    cfg = synth.get_config(args.config)
    if args.separate_critic:
        cfg = cfg.with_(separate_critic=True)
    if rank != 0:
        return
    import oracle
    cores = host_cores()
    per_step = max(0.2, 150.0 / max(1, args.steps + args.warmup))
    params = synth.make_params(cfg, 0)
    nx = dict(epochs=max(1, args.epochs), minibatches=max(1, args.minibatches),
              value_clip=args.value_clip, max_grad_norm=args.max_grad_norm)
    _, _, Bp, _ = time_oracle(cfg, per_step, cores, params, nx)
    c, b = oracle_sample(cfg, Bp)
    for _ in range(args.warmup):
        oracle.ppo_step(c, params, [b], apply=True, threads=cores, **nx)
    t0 = time.perf_counter()
    for k in range(args.steps):
        oracle.ppo_step(c, params, [b], apply=True, t=k + 1, threads=cores, **nx)
    dt = time.perf_counter() - t0
    value = b["n"] * args.steps / dt
    sample = (f"{cfg.name}-shaped T={cfg.T}, B'={Bp * cfg.agents} columns ({b['n']} samples) per "
              f"step, full network, GAE+norm+loss/grad+Adam, C double, {cores} threads on {cpu_model()}")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": cfg.name, "T": cfg.T, "B_per_step": Bp * cfg.agents, **nx},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# ------------------------------------------------------------------ roofline helpers
def load_peaks():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def kernel_table(recs, Kp, prof_ms):
    """Per-kernel rows from the profiled region; tensor fractions against the BURST bf16 peak
    (each GEMM launch is tens of microseconds: a burst, B200_PROFILING.md), HBM against copy."""
    hbm, tf_burst, _, _ = load_peaks()
    agg = {}
    for name, t, fl, by in recs:
        a = agg.setdefault(name, [0.0, 0, 0.0, 0.0])
        a[0] += t; a[1] += 1; a[2] += fl; a[3] += by
    rows = []
    for name, (t, cnt, fl, by) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        avg = t / max(cnt, 1)
        row = {"name": name, "ms_per_step": t / Kp, "share": (t / Kp) / prof_ms, "launches_per_step": cnt / Kp}
        if fl > 0:
            tfl = fl / cnt / (avg * 1e-3) / 1e12
            row.update(tflops=tfl, frac_tensor=tfl / tf_burst)
        if by > 0:
            gbs = by / cnt / (avg * 1e-3) / 1e9
            row.update(gbs=gbs, frac_hbm=gbs / hbm)
        rows.append(row)
    return agg, rows


def ncu_traffic(config, step_names, dname):
    """DRAM bytes per launch of kernel `dname` from the committed ncu launch list of this
    config (profiles/ncu_traffic.json, tools/ncu_summary.py): its launches are in the same
    order as one step's profiled records, so the k-th record is the k-th launch."""
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[config]
        src = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))["_source"][config]
    except Exception:
        return None, None
    labels, by = tr.get("launches", []), tr.get("dram_bytes", [])
    if len(labels) != len(step_names):
        return None, src
    for name, lab, b in zip(step_names, labels, by):
        short = {"fwd_l1": "fwd", "fwd_hidden": "fwd", "dX_hidden": "dX", "dX_head": "dX",
                 "dW_hidden": "dW", "dW_l1": "dW", "dW_head": "dW"}.get(name, name)
        if short != lab:
            return None, src
        if name == dname:
            return b, src
    return None, src


def roofline_of(agg, step_names=None, config=None):
    """The dominant kernel (by time; not the exchange) under the roof its algorithmic intensity
    puts it: tensor above the ridge (burst peak / copy bandwidth), else HBM."""
    hbm, tf_burst, _, src = load_peaks()
    dname, (dt, dcnt, dfl, dby) = max(((k, v) for k, v in agg.items() if k not in ("allreduce", "stats")),
                                      key=lambda kv: kv[1][0])
    davg_s = dt / dcnt * 1e-3
    traffic, tsrc = (None, None)
    if step_names:
        traffic, tsrc = ncu_traffic(config, step_names, dname)
    ridge = tf_burst * 1e12 / (hbm * 1e9)
    ai = dfl / dby if dby > 0 else float("inf")
    if dfl > 0 and ai >= ridge:
        achieved = dfl / dcnt / davg_s / 1e12
        r = {"bound": "tensor", "kernel": dname, "achieved": achieved, "peak": tf_burst,
             "unit": "TFLOP/s", "frac": achieved / tf_burst, "traffic": traffic,
             "peak_source": f"{src} bf16_tflops (burst; fp16 dense = bf16 dense, nominal ratio 1)"}
    else:
        achieved = dby / dcnt / davg_s / 1e9
        r = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm,
             "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
             "peak_source": f"{src} hbm_gbs (copy)"}
    r.update(flops_per_launch=dfl / dcnt, bytes_per_launch=dby / dcnt, intensity_flop_per_byte=ai,
             ridge_flop_per_byte=ridge, ms_per_launch=davg_s * 1e3,
             traffic_source=(f"profiles/{tsrc} (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                             f"of this launch)") if traffic is not None else None)
    return r


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
    scaling = args.scaling or ("strong" if world > 1 else "weak")

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

    nccl_id = None
    if world > 1:
        from paper_2306_16688_b200.dist import broadcast_unique_id
    import dataclasses

    def make_ctx(cfg, n):
        uid = broadcast_unique_id(device=dev) if world > 1 else None
        spec = dataclasses.replace(P.NetSpec.from_config(cfg), epochs=args.epochs,
                                   minibatches=args.minibatches, value_clip=args.value_clip,
                                   max_grad_norm=args.max_grad_norm)
        ctx = P.PPOContext(spec, max_local_n=n, rank=rank, world=world, nccl_id=uid, device=local)
        ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).to(dev))
        return ctx

    def timed(step, K, W):
        for _ in range(W):
            step()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            step()
        b.record()
        barrier()
        return max_over_ranks(a.elapsed_time(b))

    def profiled(ctx, step, Kp):
        ctx.prof_reset()
        ctx.profile(True)
        ms = timed(step, Kp, 0) / Kp
        ctx.profile(False)
        return ms, ctx.prof_records()

    cfg = synth.get_config(args.config)
    if args.separate_critic:
        cfg = cfg.with_(separate_critic=True)
    # strong: the config's batch is the GLOBAL batch, split B/K over the ranks (C-A16);
    # weak: every rank holds a full config-sized shard (the global batch grows with K)
    gcfg = cfg if scaling == "strong" else cfg.with_(B=cfg.B * world)
    b = synth.make_batch(gcfg, seed=0, world=world, rank=rank)
    b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
    n = b["n"]
    N = n * world
    keys = ("rewards", "values", "dones", "obs", "actions", "logp_old")
    host = {k: torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys}
    d = {k: host[k].to(dev) for k in keys}
    h2d_bytes = sum(host[k].numel() * host[k].element_size() for k in keys)
    ctx = make_ctx(cfg, n)
    stats = torch.zeros(P.srl.STATS_BYTES, dtype=torch.uint8, device=dev)
    stats_host = torch.zeros(P.srl.STATS_BYTES, dtype=torch.uint8).pin_memory()

    def step():
        # one C-ABI call: GAE -> global normalisation -> forward/loss/backward -> allreduce -> Adam
        ctx.train_step(N, d["rewards"], d["values"], d["dones"], d["obs"], d["actions"],
                       d["logp_old"], stats=stats)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    sampler = ClockSampler(range(world)) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    # ---------------- timed region: device-resident inputs (working set > L2: see config)
    K = args.steps
    wall0 = time.monotonic()
    h0 = time.perf_counter()
    ms_total = timed(step, K, 0)
    host_ms = (time.perf_counter() - h0) * 1e3 / K
    wall1 = time.monotonic()
    stats_dev = P.decode_stats(stats)
    # ---------------- profiled region: an event pair around every launch (serialises them)
    Kp = min(K, 100)
    prof_ms, recs = profiled(ctx, step, Kp)

    # ---------------- end to end through the pre-fetch slots (NEXT-1, §4.1): every
    # step's batch goes host (pinned) -> device inside the timed region, the upload of batch
    # k+1 on the context's copy stream overlapping the step on batch k; stats copied back
    Ke = args.e2e_steps or min(K, 100)
    hb = [host[k] for k in keys]

    def e2e_run(overlap):
        ctx.upload(0, *hb)
        ctx.train_step_slot(0, N, stats=stats)
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record()
        ctx.upload(0, *hb)
        for j in range(Ke):
            if overlap and j + 1 < Ke:
                ctx.upload((j + 1) % 2, *hb)
            ctx.train_step_slot(j % 2 if overlap else 0, N, stats=stats)
            stats_host.copy_(stats, non_blocking=True)
            if not overlap and j + 1 < Ke:
                torch.cuda.current_stream().synchronize()   # no pre-fetch: upload after the step
                ctx.upload(0, *hb)
        x1.record()
        barrier()
        return max_over_ranks(x0.elapsed_time(x1))

    e2e_ms = e2e_run(True)
    e2e_serial_ms = e2e_run(False)      # ablation (§5.3.4, E14): pre-fetching off
    # ---------------- NEXT-2: policy-worker batched inference on the same observations
    Ki = min(K, 100)
    inf_out = (torch.empty((n, len(cfg.heads)), dtype=torch.int32, device=dev),
               torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.float32, device=dev))
    seed_box = [0]

    def roll():
        seed_box[0] += 1
        ctx.rollout(d["obs"], seed=seed_box[0], actions=inf_out[0], logp=inf_out[1], value=inf_out[2])

    inf_ms = timed(roll, Ki, 3) / Ki
    if sampler:
        time.sleep(0.1)
        sampler.stop()
    comm_path = ctx.comm_path
    ctx.close()
    del d

    # ---------------- the other scaling mode (multi-GPU): same config, same code
    alt = None
    if world > 1 and not args.no_alt_scaling:
        other = "weak" if scaling == "strong" else "strong"
        acfg = cfg if other == "strong" else cfg.with_(B=cfg.B * world)
        ab = synth.make_batch_device(acfg, dev, seed=0, world=world, rank=rank)
        actx = make_ctx(cfg, ab["n"])
        An = ab["n"] * world
        ams = timed(lambda: actx.train_step(An, ab["rewards"], ab["values"], ab["dones"], ab["obs"],
                                            ab["actions"], ab["logp_old"]), K, max(3, args.warmup))
        alt = {"scaling": other, "value": An * K / (ams * 1e-3), "unit": UNIT,
               "ms_per_step": ams / K, "samples_per_step": An,
               "inputs": "device-side synthetic (synth.make_batch_device)"}
        actx.close()
        del ab

    # ---------------- every other BASELINE config on this GPU (N = 1 only): samples/s + roofline
    others = {}
    if world == 1 and not args.no_all_configs:
        plan = {"tiny": (300, 100), "atari": None, "gfootball": (30, 20), "smac": (5, 3), "hns": (3, 2)}
        for name, kk in plan.items():
            if kk is None or name == cfg.name:
                continue
            c = synth.get_config(name)
            cb = synth.make_batch_device(c, dev, seed=0)
            cctx = make_ctx(c, cb["n"])
            cs = lambda: cctx.train_step(cb["n"], cb["rewards"], cb["values"], cb["dones"], cb["obs"],
                                         cb["actions"], cb["logp_old"])
            cms = timed(cs, kk[0], 2)
            pms, crecs = profiled(cctx, cs, kk[1])
            cagg, _ = kernel_table(crecs, kk[1], pms)
            others[name] = {"value": cb["n"] * kk[0] / (cms * 1e-3), "unit": UNIT,
                            "ms_per_step": cms / kk[0], "steps": kk[0], "samples_per_step": cb["n"],
                            "roofline": roofline_of(cagg),
                            "inputs": "device-side synthetic (synth.make_batch_device)"}
            cctx.close()
            del cb
            torch.cuda.empty_cache()

    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    import math
    agg, kernels = kernel_table(recs, Kp, prof_ms)
    nper = len(recs) // max(Kp, 1)
    step_names = [r[0] for r in recs[:nper] if not (r[0] == "allreduce" and comm_path == "nccl")]
    roofline = roofline_of(agg, step_names=step_names, config=cfg.name)
    # our kernels per step: every launch srl_ppo_train_step makes is one profiled record
    # (the profiling region runs the same steps); NCCL's allreduce is not ours
    ours = sum(1 for r in recs if not (r[0] == "allreduce" and comm_path == "nccl"))
    per_step = ours / Kp
    L = len(cfg.hidden)
    updates = max(1, args.epochs) * max(1, args.minibatches)
    # the oracle baseline on the host cores: rank 0 at N = 1 only (the contract)
    cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baselines(cfg, args.cpu_seconds)
    clocks = sampler.summary(wall0, wall1) if sampler else None
    out = {
        "metric": METRIC, "value": N * K / (ms_total * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": max(3, args.warmup), "ms_per_step": ms_total / K, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f16",
        "data": "synthetic",
        "config": {"workload": cfg.name, "T": cfg.T, "B_global": N // cfg.T, "B_per_rank": n // cfg.T,
                   "obs_dim": cfg.obs_dim,
                   "hidden": list(cfg.hidden), "heads": list(cfg.heads), "samples_per_step": N,
                   "frames_per_step": N * cfg.frame_skip, "parallelism": f"dp{world}",
                   "grad_allreduce": comm_path,
                   "epochs": max(1, args.epochs), "minibatches": max(1, args.minibatches),
                   "value_clip": args.value_clip, "max_grad_norm": args.max_grad_norm,
                   "separate_critic": bool(args.separate_critic),
                   "l2": "no flush: per-step working set > L2 (obs %.0f MB + activations %.0f MB + "
                         "dZ %.0f MB per rank vs 126 MB L2)" % (
                             n * cfg.ld_obs * 2 / 1e6, n * sum(cfg.hidden) * 2 / 1e6,
                             n * max(cfg.hidden) * 4 / 1e6)},
        "frames_per_s": N * cfg.frame_skip * K / (ms_total * 1e-3),
        "sample_updates_per_s": N * updates * K / (ms_total * 1e-3),
        "host_submit_ms_per_step": host_ms,
        "profiled_ms_per_step": prof_ms,
        "e2e": {"value": N * Ke / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d_bytes * world,
                "d2h_bytes_per_step": P.srl.STATS_BYTES * world, "steps": Ke,
                "no_prefetch": {"value": N * Ke / (e2e_serial_ms * 1e-3), "unit": UNIT,
                                "what": "ablation: upload after each step, no overlap (PAPER.md §5.3.4)"}},
        "gpu_launches": int(round(per_step * K)),
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
    if alt:
        out["alt_scaling"] = alt
    if others:
        out["configs"] = others
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
