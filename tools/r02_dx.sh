python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_head_fused.py tests/test_gpu_ac.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-all-configs > gpurun_out/hf_bench.json 2> gpurun_out/hf_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/hf_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), " ".join(f'{k["name"]}={k["ms_per_step"]*1e3:.1f}' for k in d["kernels"]))
PY
timeout 300 ncu --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python tools/kernel_probe.py step atari 2 2>&1 | grep -E "gemm_tc|gpu__time|dram__"
