# fused exchange check (gpurun --gpus 2 or 4): multi-GPU tests, then the bench at N = GPUs with
# the fused launch and with SRL_XFUSED=0
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider 2>&1 | tail -2
for x in 1 0; do
SRL_XFUSED=$x timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$x bench.py --gpus $N --steps 200 --warmup 10 > gpurun_out/x_bench_$x.json 2> gpurun_out/x_bench_$x.err
python - $x <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/x_bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("XFUSED", sys.argv[1], d["scaling"], "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), "alt", round(d["alt_scaling"]["value"]/1e6, 1), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done
