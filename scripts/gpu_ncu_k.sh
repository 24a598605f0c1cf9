#!/bin/bash
# ncu --set full captures of the kernels named in $KS (space separated regexes), one report each
mkdir -p gpurun_out
TAG=${1:-k}
for K in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-3} -c 1 -o gpurun_out/${TAG}_${K} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG}_${K}.log 2>&1
  tail -1 gpurun_out/${TAG}_${K}.log
done
