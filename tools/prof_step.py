"""Run a few Atari-shaped srl_ppo_train_step calls (for ncu captures of single kernels).

    ncu --set full -k regex:gemm_tc_kernel --launch-skip 20 --launch-count 1 \
        python tools/prof_step.py        # 5th GEMM (dX_head) of the 3rd step
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "atari")
b = synth.make_batch(cfg, seed=0)
b["logp_old"] = synth.logp_old_uniform_policy(cfg, b["xi"])
d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda()
     for k in ("rewards", "values", "dones", "obs", "actions", "logp_old")}
ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).cuda())
for _ in range(4):
    ctx.train_step(b["n"], d["rewards"], d["values"], d["dones"], d["obs"], d["actions"], d["logp_old"])
torch.cuda.synchronize()
print("ok")
