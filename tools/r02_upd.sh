python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_next3.py tests/test_gpu_ac.py tests/test_gpu_exchange.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in atari gfootball; do
timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/hf_bench.json 2> gpurun_out/hf_bench.err
python - $c <<'PY'
import json, sys
d = json.loads(open("gpurun_out/hf_bench.json").read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done
