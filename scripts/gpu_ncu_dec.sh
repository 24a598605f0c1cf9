#!/bin/bash
# ncu --set full of the decoder's kernels: $2 = cfg2 (bench step) or cfg5 (one slab)
mkdir -p gpurun_out
TAG=${1:-nd}; WL=${2:-cfg2}
if [ "$WL" = cfg2 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tfd_maps|k_tfd_emit|k_tfd_count" -s 6 -c 3 -o gpurun_out/${TAG}_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg2.log 2>&1
else
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tfd_maps|k_tfd_emit|k_tfd_count" -s 3 -c 3 -o gpurun_out/${TAG}_cfg5 \
    python scripts/tfd_probe.py cfg5slab > gpurun_out/${TAG}_cfg5.log 2>&1
fi
ls -la gpurun_out/*.ncu-rep
