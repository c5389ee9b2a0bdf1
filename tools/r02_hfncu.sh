# one ncu --set full capture of head_fused at the Atari shape (after a plain run exits 0)
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 120 python tools/kernel_probe.py step atari 2 > gpurun_out/hf_probe.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:head_fused --launch-skip 1 --launch-count 1 -f -o gpurun_out/${1:-r02_hf3} python tools/kernel_probe.py step atari 2 > gpurun_out/hf_ncu.log 2>&1
tail -2 gpurun_out/hf_ncu.log
