python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
for lib in paper_2306_16688_b200/libsrl.so variants/gae32/libsrl.so variants/gae8/libsrl.so; do
for c in atari smac hns gfootball; do
  SRL_LIB=$lib timeout 300 ncu --clock-control none -k regex:gae_kernel -s 1 -c 1 --metrics gpu__time_duration.sum python tools/kernel_probe.py gae $c 2 2>&1 | grep -E "gpu__time" | sed "s|^|$(echo $lib | cut -d/ -f2) $c |"
done; done
