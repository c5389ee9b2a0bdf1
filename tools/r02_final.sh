# round-end confirmation (gpurun --gpus 2): smoke(), the whole GPU suite (multi-GPU tests at 2
# ranks), the default bench line, the reference (oracle) arm, a 2-GPU bench.  -> gpurun_out/r02z_*
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02z_smoke.txt 2>&1; tail -1 gpurun_out/r02z_smoke.txt
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02z_gpu_tests.txt 2>&1; tail -1 gpurun_out/r02z_gpu_tests.txt
timeout 600 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02z_bench_ref.json 2> gpurun_out/r02z_bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/r02z_bench_n2.json 2> gpurun_out/r02z_bench_n2.err
python - <<'PY'
import json
for f in ["r02z_bench.json", "r02z_bench_ref.json", "r02z_bench_n2.json"]:
    try:
        d = json.loads(open("gpurun_out/" + f).read().strip().splitlines()[-1])
        print(f, d.get("impl", "ours"), d.get("n_gpus"), round(d["value"] / 1e6, 3), "M/s", d.get("ms_per_step"), "frac", (d.get("roofline") or {}).get("frac"), "e2e", (d.get("e2e") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
