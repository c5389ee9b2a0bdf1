# A/B of env switches on the 1-GPU Atari bench: "$@" = list of "NAME=VAL[,NAME=VAL]" settings
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
for cfg in "$@"; do
  env $(echo "$cfg" | tr ',' ' ') timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done
