#!/bin/bash
# ncu --set full capture of the kernels matching $2 (first $3 matches after the warm-up).
mkdir -p gpurun_out
TAG=$1; KREGEX=$2; CNT=${3:-3}; SKIP=${4:-0}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP} -c ${CNT} -o gpurun_out/${TAG}_prof \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_prof.log 2>&1
tail -3 gpurun_out/${TAG}_prof.log
