"""Phase marks of update_kernel (variant build with -DSRL_UPD_TRACE):

    python tools/build_variant.py updtrace SRL_UPD_TRACE
    SRL_LIB=variants/updtrace/libsrl.so python tools/upd_trace.py atari

Runs the train step, then prints per phase the mean / max over blocks of the ns (globaltimer) since the
earliest block's start mark (0 start, 1 after griddep_wait, 2 weights finalised, 3 biases +
stats, 4 after the grid barrier, 5 Adam done)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
from paper_2306_16688_b200 import srl  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "atari"
cfg = synth.get_config(name)
dev = torch.device("cuda", 0)
b = synth.make_batch_device(cfg, dev, seed=0)
ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).to(dev))
fn = srl.lib().srl_debug_upd_trace
fn.argtypes = [ctypes.c_void_p]
buf = np.zeros(256 * 12, dtype=np.int64)
for _ in range(4):
    ctx.train_step(b["n"], b["rewards"], b["values"], b["dones"], b["obs"], b["actions"], b["logp_old"])
torch.cuda.synchronize()
fn(buf.ctypes.data)
t = buf.reshape(256, 12)[:148].astype(np.float64)
t0 = t[:, 0].min()
for k, nm in [(0, "start"), (1, "griddep_wait"), (2, "weights"), (6, "weight warp items"),
              (7, "biases"), (3, "stats"), (4, "barrier"), (5, "adam")]:
    x = t[:, k] - t0
    print(f"{nm:14s} mean {x.mean():9.0f}  max {x.max():9.0f}  min {x.min():9.0f}")
