#!/bin/bash
# A/B of library variants: tools/ab.sh <variant dirs...> ("base" = in-tree build); 2 runs each
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="variants/$v/libsrl.so"; fi
  SRL_LIB=$lib python bench.py --steps 200 --warmup 10 --no-cpu-baseline $BENCH_ARGS > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python tools/ab_show.py $v gpurun_out/ab_$v.json
done
done
