python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_next3.py tests/test_gpu_head_fused.py -q -x -p no:cacheprovider 2>&1 | tail -1
for v in updtrace updoldtrace; do echo "== $v"; SRL_LIB=variants/$v/libsrl.so python tools/upd_trace.py atari | tail -8; done
for i in 1 2; do
for lib in paper_2306_16688_b200/libsrl.so variants/updold/libsrl.so; do
  SRL_LIB=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - $lib <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1].split("/")[-2], "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
done; done
