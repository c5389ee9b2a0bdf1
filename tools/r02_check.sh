# 2-GPU check after an update/stats/exchange change (gpurun --gpus 2): the single-GPU suites
# that cover the step, the exchange tests, then the bench at N=1 and N=2
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02c_gpu.txt 2>&1
tail -3 gpurun_out/r02c_gpu.txt
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r02c_bench_n1.json 2> gpurun_out/r02c_bench_n1.err
tail -c 600 gpurun_out/r02c_bench_n1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 10 > gpurun_out/r02c_bench_n2.json 2> gpurun_out/r02c_bench_n2.err
tail -c 600 gpurun_out/r02c_bench_n2.json
