"""Run a few srl_ppo_train_step calls of a config (for ncu captures of single kernels and for
localising faults: with CUDA_LAUNCH_BLOCKING=1 the failing launch's srl_* error names it).

    python tools/prof_step.py [config] [B] [steps]
    ncu --set full -k regex:head_fused -s 2 -c 1 python tools/prof_step.py atari
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "atari")
if len(sys.argv) > 2:
    cfg = cfg.with_(B=int(sys.argv[2]))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
b = synth.make_batch(cfg, seed=0)
b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda()
     for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}
ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).cuda())
t0 = time.time()
try:
    for k in range(steps):
        st = ctx.train_step(b["n"], d["rewards"], d["values"], d["dones"], d["obs"], d["actions"],
                            d["logp_old"])
        if os.environ.get("CUDA_LAUNCH_BLOCKING") == "1":
            torch.cuda.synchronize()
            print(f"step {k} ok", P.decode_stats(st)["loss"], flush=True)
    torch.cuda.synchronize()
except Exception as e:
    print(f"FAILED after {time.time() - t0:.1f} s: {e}", flush=True)
    raise
print(f"ok ({time.time() - t0:.2f} s)")
