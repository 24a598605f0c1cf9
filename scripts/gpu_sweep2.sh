#!/bin/bash
# variants: cfg2 bench phases + cfg5 slab probe + decode parity subset
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  MGRC_NVCC_EXTRA="$V" python paper_2401_05994_b200/build.py --force > /dev/null 2>&1 || { echo "build [$V] failed"; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYK:-container_parity or slab or fuzz}" > gpurun_out/sw2_${i}_pytest.log 2>&1; tail -1 gpurun_out/sw2_${i}_pytest.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw2_$i.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw2_$i.json')); p=d['phases_ms_per_step']
print('[$V] cfg2', round(d['value'],1), round(d['decompress_gbs'],1), p['huff_sync']['ms'])" 2>/dev/null || echo "[$V] cfg2 bench failed"
  timeout 300 python scripts/phase_probe.py 256 2>/dev/null | grep decompress | sed "s/^/[$V] slab /"
done
