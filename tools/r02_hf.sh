# fused-head iteration (gpurun, 1 GPU): head tests, per-role trace, bench at N=1
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_head_fused.py -q -x -p no:cacheprovider > gpurun_out/hf_tests.txt 2>&1
tail -2 gpurun_out/hf_tests.txt
for c in atari gfootball; do SRL_LIB=variants/hftrace/libsrl.so timeout 120 python tools/hf_trace.py $c 5; done > gpurun_out/hf_trace.txt 2>&1
cat gpurun_out/hf_trace.txt
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/hf_bench.json 2> gpurun_out/hf_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/hf_bench.json").read().strip().splitlines()[-1])
print("value", d["value"] / 1e6, "ms", d["ms_per_step"], "e2e", d["e2e"]["value"] / 1e6)
for k in d["kernels"]: print("  ", k["name"], round(k["ms_per_step"] * 1e3, 1))
PY
