# multi-GPU confirmation (gpurun --gpus 4): exchange tests at 2 and 4 ranks, then the bench at
# N = 2 and 4 (strong scaling by default, weak in alt_scaling), fused peer path and NCCL;
# gFootball (the BASELINE's 1/2/4/8-GPU config) at N = 1, 2, 4.  Outputs gpurun_out/${TAG}_*.
TAG=${TAG:-r02f}
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/${TAG}_gpu_multi.txt 2>&1
tail -1 gpurun_out/${TAG}_gpu_multi.txt
run() {  # run <N> <out> [env...] -- bench args
  local n=$1 out=$2; shift 2
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n $BENCH_ARGS > gpurun_out/${TAG}_$out.json 2> gpurun_out/${TAG}_$out.err
}
for n in 2 4; do
  BENCH_ARGS="--steps 200 --warmup 10" run $n bench_n$n SRL_XFUSED=1
  BENCH_ARGS="--steps 200 --warmup 10 --no-alt-scaling" run $n bench_n${n}_nccl SRL_P2P_AR=0
done
for n in 2 4; do BENCH_ARGS="--config gfootball --steps 50 --warmup 5" run $n bench_n${n}_gf SRL_XFUSED=1; done
timeout 300 python bench.py --config gfootball --steps 50 --warmup 5 --no-all-configs --no-cpu-baseline > gpurun_out/${TAG}_bench_n1_gf.json 2> gpurun_out/${TAG}_bench_n1_gf.err
python - $TAG <<'PY'
import json, sys, glob
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["config"]["workload"], d["n_gpus"], d["scaling"], round(d["value"] / 1e6, 1), "M/s", round(d["ms_per_step"], 4), "ms", "alt", round(d.get("alt_scaling", {}).get("value", 0) / 1e6, 1))
    except Exception as e:
        print(f, "ERR", e)
PY
