"""Diagnostic: gradient error vs distance of rho from the clip kinks (HnS/SMAC reduced)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle, synth
from ppo_harness import gpu_step, grad_errors, make_inputs

for name, B in (("hns", 16), ("smac", 200), ("atari", 16)):
    base = synth.get_config(name).with_(B=B)
    for clip, margin in ((0.2, 0.0), (0.2, 0.01), (0.2, 0.03), (10.0, 0.0)):
        cfg = base.with_(clip_eps=clip)
        params, b = make_inputs(cfg, seed=11)
        lp = oracle.log_pi(cfg, params, b["obs"], b["actions"])
        xi = lp - b["logp_old"]
        if margin > 0:
            for k in (np.log(1 + clip), np.log(1 - clip)):
                close = np.abs(xi - k) < margin
                xi[close] = k + np.sign(xi[close] - k + 1e-30) * margin
            b["logp_old"] = (lp - xi).astype(np.float32)
        g = gpu_step(cfg, params, [b], apply=False)
        o = oracle.ppo_step(cfg, params, [b], apply=False)
        e = grad_errors(cfg, g["bucket"][:cfg.n_params], o["grad"])
        worst = max(e.items(), key=lambda kv: kv[1][0])
        print(f"{name} clip={clip} margin={margin}: worst {worst[0]} relL2={worst[1][0]:.2e} maxrel={worst[1][1]:.2e}; "
              f"clipfrac gpu={g['stats']['clip_fraction']:.5f} ref={o['sums'][3]/o['N']:.5f}", flush=True)
