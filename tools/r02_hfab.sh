# A/B of a head_fused build variant: head_fused DRAM bytes + duration and the Atari bench
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
for lib in paper_2306_16688_b200/libsrl.so "$@"; do
  echo "== $lib"
  SRL_LIB=$lib timeout 300 ncu --clock-control none -k regex:head_fused -s 1 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python tools/kernel_probe.py step atari 2 2>&1 | grep -E "gpu__time|dram__"
  SRL_LIB=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print("value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done
