# fused-head tests, then one ncu --set full capture of head_fused at the Atari shape
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_head_fused.py tests/test_gpu_ppo.py tests/test_gpu_ac.py tests/test_gpu_next3.py -q -x -p no:cacheprovider > gpurun_out/hf_tests.txt 2>&1
tail -2 gpurun_out/hf_tests.txt
timeout 120 python tools/kernel_probe.py step atari 2 > gpurun_out/hf_probe.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:head_fused --launch-skip 1 --launch-count 1 -f -o gpurun_out/r02_hf2 python tools/kernel_probe.py step atari 2 > gpurun_out/hf_ncu.log 2>&1
tail -3 gpurun_out/hf_ncu.log
