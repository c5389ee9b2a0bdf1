# multi-GPU confirmation (gpurun --gpus 4): exchange tests at 2 and 4 ranks, then the bench at
# N = 2 and 4 (strong scaling by default, weak in alt_scaling), peer-memory path and NCCL
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
nvidia-smi topo -m > gpurun_out/r02_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/r02_gpu_multi.txt 2>&1
tail -3 gpurun_out/r02_gpu_multi.txt
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 200 --warmup 10 > gpurun_out/r02_bench_n$n.json 2> gpurun_out/r02_bench_n$n.err
  SRL_P2P_AR=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 200 --warmup 10 --no-alt-scaling > gpurun_out/r02_bench_n${n}_nccl.json 2> gpurun_out/r02_bench_n${n}_nccl.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config gfootball --steps 50 --warmup 5 > gpurun_out/r02_bench_n4_gf.json 2> gpurun_out/r02_bench_n4_gf.err
timeout 300 python bench.py --config gfootball --steps 50 --warmup 5 --no-all-configs --no-cpu-baseline > gpurun_out/r02_bench_n1_gf.json 2> gpurun_out/r02_bench_n1_gf.err
ls gpurun_out
