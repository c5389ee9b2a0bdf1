"""Per-role wait accounting of head_fused_kernel (variant build with -DSRL_HF_TRACE):

    python tools/build_variant.py hftrace SRL_HF_TRACE
    SRL_LIB=variants/hftrace/libsrl.so python tools/hf_trace.py atari

Runs the train step `reps` times and prints, per slot, the mean over CTAs of the cycles per
launch (clock64; slot meanings in head_fused.cu under SRL_HF_TRACE)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
from paper_2306_16688_b200 import srl  # noqa: E402
import synth  # noqa: E402

NAMES = {0: "pass-A issuer loop", 1: "prodA wait emptyA", 2: "prodB wait emptyB",
         3: "loss wait lfull (tile 0)", 4: "mmaA wait lempty", 5: "mmaB wait gfull", 6: "mmaA wait fullA",
         7: "mmaB wait dempty/fullB", 8: "loss wait lfull (rest)", 9: "loss wait gempty", 10: "loss loop end",
         11: "dtanh wait dfull", 12: "dtanh wait fullB", 13: "dtanh pair barrier",
         14: "dtanh staging acquire", 15: "dtanh loop end"}
name = sys.argv[1] if len(sys.argv) > 1 else "atari"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.get_config(name)
dev = torch.device("cuda", 0)
b = synth.make_batch_device(cfg, dev, seed=0)
ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"])
ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).to(dev))
fn = srl.lib().srl_debug_hf_trace
fn.argtypes = [ctypes.c_void_p]
buf = np.zeros(256 * 16, dtype=np.uint64)
step = lambda: ctx.train_step(b["n"], b["rewards"], b["values"], b["dones"], b["obs"],
                              b["actions"], b["logp_old"])
step()
torch.cuda.synchronize()
fn(buf.ctypes.data)
for _ in range(reps):
    step()
torch.cuda.synchronize()
fn(buf.ctypes.data)
t = buf.reshape(256, 16)[:148].astype(np.float64) / reps
m_tiles = (b["n"] + 127) // 128
print(f"{name}: n = {b['n']}, {m_tiles} tiles over 148 CTAs; cycles per launch, mean (max) over CTAs")
for k in range(16):
    print(f"  {k:2d} {NAMES[k]:24s} {t[:, k].mean():10.0f} ({t[:, k].max():10.0f})")
