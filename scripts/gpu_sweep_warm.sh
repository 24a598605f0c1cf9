#!/bin/bash
# warm-up length sweep of the sync pass (cfg2 phases)
mkdir -p gpurun_out
for W in ${WARMS:-256 384 512 768 1024}; do
  MGRC_NVCC_EXTRA="-DMGRC_WARM_BITS=$W" python paper_2401_05994_b200/build.py --force > /dev/null 2>&1 || { echo "build $W failed"; continue; }
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/warm_$W.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/warm_$W.json')); p=d['phases_ms_per_step']
print($W, round(d['value'],1), round(d['decompress_gbs'],1), {k: v['ms'] for k, v in p.items() if k.startswith('huff')})"
done
