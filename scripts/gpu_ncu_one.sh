#!/bin/bash
# ncu --set full of one kernel launch (regex $2) from the bench (workload $3 optional)
mkdir -p gpurun_out
TAG=${1:-n}; K=${2:-k_huff_tfd}; WL=${3:-cfg2_513cubed_f32_inf_rel1e-4}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${K} -s 3 -c 1 -o gpurun_out/${TAG} \
  python bench.py --workload ${WL} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
