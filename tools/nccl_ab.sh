#!/bin/bash
# NCCL algorithm/protocol A/B at N GPUs (weak-scaling bench): tools/nccl_ab.sh N
N=${1:-4}
mkdir -p gpurun_out
run() {
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus $N --steps 200 --warmup 10 --no-cpu-baseline \
    > gpurun_out/nccl.json 2> gpurun_out/nccl.err
  python - "$*" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/nccl.json").readline())
    ar = [k["ms_per_step"] * 1e3 for k in d["kernels"] if k["name"] in ("allreduce", "adv_norm")]
    print(sys.argv[1] or "default", round(d["value"] / 1e6, 1), "M/s", round(d["ms_per_step"] * 1e3, 1), "us  allreduce/adv_norm(prof) us", [round(x, 1) for x in ar])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
}
run NCCL_DEBUG=WARN
run NCCL_ALGO=NVLS
run NCCL_ALGO=Ring
run NCCL_ALGO=Tree
run NCCL_PROTO=LL128
run NCCL_PROTO=LL
run NCCL_PROTO=Simple
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING env python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/nccl_info.err
grep -i "nvls\|algo\|proto" gpurun_out/nccl_info.err | head -20
