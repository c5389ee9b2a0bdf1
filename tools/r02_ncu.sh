# ncu evidence for profiles/ (1 GPU): the launch list of one Atari step, full captures of the
# step's kernels, the GAE scan at SMAC / HnS and the update launch at HnS
python -m paper_2306_16688_b200.build > gpurun_out/build.log 2>&1
P="ncu --clock-control none"
F="$P --set full --import-source on"
python tools/prof_step.py atari 1024 6 > gpurun_out/plain.log 2>&1 && \
  $P --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r02_launches.csv python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
$F -k regex:head_fused -s 2 -c 1 -o gpurun_out/r02_head_fused python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
$F -k regex:update_kernel -s 2 -c 1 -o gpurun_out/r02_update python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
# gemm launches per step: fwd_l1, fwd_hidden, dW_hidden, dX_hidden, dW_l1 (step 2 = launches 10..14)
$F -k regex:gemm_tc_kernel -s 11 -c 1 -o gpurun_out/r02_fwd_hidden python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
$F -k regex:gemm_tc_kernel -s 12 -c 1 -o gpurun_out/r02_dW_hidden python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
$F -k regex:gemm_tc_kernel -s 13 -c 1 -o gpurun_out/r02_dX_hidden python tools/prof_step.py atari 1024 6 > /dev/null 2>&1
for c in smac hns; do
  python tools/kernel_probe.py gae $c > gpurun_out/probe_gae_$c.log 2>&1 && \
    $F -k regex:gae_kernel -s 2 -c 1 -o gpurun_out/r02_gae_$c python tools/kernel_probe.py gae $c > /dev/null 2>&1
done
python tools/kernel_probe.py step hns 2 > gpurun_out/probe_step_hns.log 2>&1 && \
  $F -k regex:update_kernel -s 1 -c 1 -o gpurun_out/r02_update_hns python tools/kernel_probe.py step hns 2 > /dev/null 2>&1
ls gpurun_out | grep -c ncu-rep
