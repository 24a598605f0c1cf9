#!/bin/bash
# Build variants (MGRC_NVCC_EXTRA flag sets separated by ';' in $VARIANTS), for each: decode parity subset + cfg2 phases
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  MGRC_NVCC_EXTRA="$V" python paper_2401_05994_b200/build.py --force > /dev/null 2>&1 || { echo "build [$V] failed"; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYK:-container_parity or slab}" > gpurun_out/sw_${i}_pytest.log 2>&1; tail -1 gpurun_out/sw_${i}_pytest.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/sw_$i.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw_$i.json')); p=d['phases_ms_per_step']
print('[$V]', round(d['value'],1), round(d['compress_gbs'],1), round(d['decompress_gbs'],1), {k: v['ms'] for k, v in p.items()})"
done
