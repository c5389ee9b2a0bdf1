"""Diagnose a two-trunk second step: per-tensor errors of step 2's gradient vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from ppo_harness import gpu_step, grad_errors, make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hns"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
sep = len(sys.argv) <= 3 or sys.argv[3] == "1"
cfg = synth.get_config(name).with_(B=B, separate_critic=sep)
params, b = make_inputs(cfg, seed=53)
g = gpu_step(cfg, params, [b], apply=True)
o1 = oracle.ppo_step(cfg, params, [b], apply=False)
e1 = grad_errors(cfg, g["bucket"][:cfg.n_params], o1["grad"])
p1 = g["params"].astype(np.float32)
g2 = gpu_step(cfg, params, [b], apply=False, ctx=g["ctx"])
o2 = oracle.ppo_step(cfg, p1, [b], apply=False)
e2 = grad_errors(cfg, g2["bucket"][:cfg.n_params], o2["grad"])
for k in e1:
    print(f"{k:5s} step1 {e1[k][0]:.2e} {e1[k][1]:.2e}   step2 {e2[k][0]:.2e} {e2[k][1]:.2e}")
