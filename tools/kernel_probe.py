"""Run one kernel family at a BASELINE config's full size, for ncu captures and CUDA-event
timings of kernels whose HBM rate is only meaningful at large sizes:

    python tools/kernel_probe.py gae smac        # srl_gae over [400][20480] (5 calls)
    python tools/kernel_probe.py step hns        # srl_ppo_train_step (3 calls): update_kernel etc.

Prints the per-call CUDA-event time and the algorithmic GB/s (17 B/sample for GAE).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
import synth  # noqa: E402

what, name = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = synth.get_config(name)
dev = torch.device("cuda", 0)
b = synth.make_batch_device(cfg, dev, seed=0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if what == "gae":
    adv = torch.empty_like(b["rewards"])
    ret = torch.empty_like(b["rewards"])
    st = torch.empty(3, dtype=torch.float64, device=dev)
    for _ in range(2):
        P.gae(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam, adv, ret, st)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        P.gae(b["rewards"], b["values"], b["dones"], cfg.gamma, cfg.lam, adv, ret, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"gae {name}: {ms * 1e3:.1f} us per call, {17.0 * b['n'] / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic "
          f"(17 B/sample, n = {b['n']}; the call includes the moments merge launch)")
else:
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
    ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).to(dev))
    step = lambda: ctx.train_step(b["n"], b["rewards"], b["values"], b["dones"], b["obs"],
                                  b["actions"], b["logp_old"])
    step()
    torch.cuda.synchronize()
    ctx.prof_reset()
    ctx.profile(True)
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    ctx.profile(False)
    agg = {}
    for nm, ms, fl, by in ctx.prof_records():
        a = agg.setdefault(nm, [0.0, 0, fl, by])
        a[0] += ms
        a[1] += 1
    for nm, (ms, cnt, fl, by) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        avg = ms / cnt
        print(f"{nm:14s} {avg * 1e3:10.1f} us  {by / (avg * 1e-3) / 1e9:8.0f} GB/s  {fl / (avg * 1e-3) / 1e12:8.1f} TFLOP/s")
print("ok")
