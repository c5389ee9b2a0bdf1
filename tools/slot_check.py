"""NEXT-1 slot path vs device path, step by step (gradients and parameters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "gfootball").with_(B=int(sys.argv[2]) if len(sys.argv) > 2 else 16)
b = synth.make_batch(cfg, seed=0)
b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
keys = ("rewards", "values", "dones", "obs", "actions", "logp_old")
host = [torch.from_numpy(np.ascontiguousarray(b[k])).pin_memory() for k in keys]
dev = [h.cuda() for h in host]
spec = P.NetSpec.from_config(cfg)
a = P.PPOContext(spec, max_local_n=b["n"])
c = P.PPOContext(spec, max_local_n=b["n"])
p0 = torch.from_numpy(synth.make_params(cfg, 0)).cuda()
a.load_params(p0)
c.load_params(p0)
mode = sys.argv[3] if len(sys.argv) > 3 else "overlap"
c.upload(0, *host)
for k in range(3):
    a.train_step(b["n"], *dev)
    if mode == "overlap":
        if k + 1 < 3:
            c.upload((k + 1) % 2, *host)
        c.train_step_slot(k % 2, b["n"])
    else:
        c.train_step_slot(0, b["n"])
        torch.cuda.synchronize()
        if k + 1 < 3:
            c.upload(0, *host)
    torch.cuda.synchronize()
    ga, gc = a.grads().cpu().numpy(), c.grads().cpu().numpy()
    print(f"step {k}: grads differ in {int(np.sum(ga != gc))} entries (max {np.abs(ga - gc).max():.3e}); "
          f"params identical {torch.equal(a.params(), c.params())}", flush=True)
