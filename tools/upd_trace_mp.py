"""update_kernel phase marks at world > 1 (variant build with -DSRL_UPD_TRACE), one line per rank:

    python tools/build_variant.py updtrace SRL_UPD_TRACE
    SRL_LIB=variants/updtrace/libsrl.so torchrun --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tools/upd_trace_mp.py atari

Each rank runs the strong-scaling shard of the config for 6 steps and prints, per phase, the
mean / max over blocks of the ns since its own launch's earliest block start (globaltimer is
per GPU, so ranks are not compared in absolute time)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2306_16688_b200 as P  # noqa: E402
from paper_2306_16688_b200 import srl  # noqa: E402
from paper_2306_16688_b200.dist import broadcast_unique_id  # noqa: E402
import synth  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
name = sys.argv[1] if len(sys.argv) > 1 else "atari"
cfg = synth.get_config(name)
cfg = cfg.with_(B=cfg.B // world)
dev = torch.device("cuda", local)
b = synth.make_batch_device(cfg, dev, seed=rank)
uid = broadcast_unique_id(device=dev)
ctx = P.PPOContext(P.NetSpec.from_config(cfg), max_local_n=b["n"], rank=rank, world=world, nccl_id=uid, device=local)
ctx.load_params(torch.from_numpy(synth.make_params(cfg, 0)).to(dev))
fn = srl.lib().srl_debug_upd_trace
fn.argtypes = [ctypes.c_void_p]
buf = np.zeros(256 * 12, dtype=np.int64)
N = b["n"] * world
for _ in range(6):
    ctx.train_step(N, b["rewards"], b["values"], b["dones"], b["obs"], b["actions"], b["logp_old"])
torch.cuda.synchronize()
fn(buf.ctypes.data)
t = buf.reshape(256, 12)[:148].astype(np.float64)
t0 = t[:, 0].min()
out = [f"rank {rank}:"]
for k, nm in [(1, "wait"), (2, "w"), (6, "wwarp"), (7, "bias"), (3, "stats"), (4, "bar1"), (8, "xchg"), (9, "bar2"), (5, "adam")]:
    x = t[:, k] - t0
    out.append(f"{nm} {x.mean() / 1e3:.1f}/{x.max() / 1e3:.1f}")
print("  ".join(out), flush=True)
dist.destroy_process_group()
