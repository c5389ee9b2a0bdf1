"""Two contexts, same inputs, N chained train steps each: are gradients / parameters bit-identical?

    python tools/determinism.py [config] [B] [steps]      (SRL_HEAD_FUSED / SRL_PDL respected)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "gfootball")
if len(sys.argv) > 2:
    cfg = cfg.with_(B=int(sys.argv[2]))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
b = synth.make_batch(cfg, seed=0)
b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda()
     for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}
res = []
for rep in range(2):
    ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
    ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).cuda())
    gs = []
    for k in range(steps):
        ctx.train_step(b["n"], d["rewards"], d["values"], d["dones"], d["obs"], d["actions"], d["logp_old"])
        gs.append(ctx.grads().cpu().numpy())
    res.append((gs, ctx.params().cpu().numpy()))
    ctx.close()
for k in range(steps):
    a, c = res[0][0][k], res[1][0][k]
    nd = int(np.sum(a != c))
    print(f"step {k}: grads differ in {nd} of {a.size} entries, max |diff| {np.abs(a - c).max():.3e}")
print("params identical:", np.array_equal(res[0][1], res[1][1]))
