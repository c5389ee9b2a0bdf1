# loss-chunk A/B: head tests, per-role trace, bench (new vs variants/lossold)
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_head_fused.py tests/test_gpu_ppo.py -q -x -p no:cacheprovider 2>&1 | tail -1
SRL_LIB=variants/hftrace/libsrl.so timeout 120 python tools/hf_trace.py atari 5 | grep -E " 8 | 9 | 10 | 11 | 15 "
for i in 1 2; do
for lib in paper_2306_16688_b200/libsrl.so variants/lossold/libsrl.so; do
  SRL_LIB=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - $lib <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1].split("/")[-2], "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done; done
for lib in paper_2306_16688_b200/libsrl.so variants/lossold/libsrl.so; do
SRL_LIB=$lib ncu --clock-control none -k regex:head_fused -s 1 -c 1 --metrics gpu__time_duration.sum python tools/kernel_probe.py step atari 2 2>&1 | grep "gpu__time" | sed "s|^|$(echo $lib | cut -d/ -f2) |"
done
