#!/bin/bash
# build-flag sweep of the fused pass (MGRC_NVCC_EXTRA variants), then one ncu capture of the default build
mkdir -p gpurun_out
TAG=${1:-sw}
VARIANTS=${VARIANTS:-"-DMGRC_FINE_MINB=5 -DMGRC_FINE_MINB=6 -DMGRC_FINE_MINB=8"}
for v in $VARIANTS; do
  MGRC_NVCC_EXTRA="$v" timeout 900 python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/${TAG}_build.log 2>&1 || { echo "build $v failed"; tail -5 gpurun_out/${TAG}_build.log; continue; }
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b.json 2>> gpurun_out/${TAG}_bench.err
  V="$v" TAG=$TAG python - <<"PY"
import json,os
d=json.loads(open(f"gpurun_out/{os.environ['TAG']}_b.json").read().strip().splitlines()[-1])
p=d["phases_ms_per_step"]
print(os.environ['V'], "c", round(d["compress_gbs"],1), "fine", p["fine"]["ms"], "pack", p["pack"]["ms"])
PY
done
if [ -n "$NCU_K" ]; then
  timeout 900 python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/${TAG}_build.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_K} -s 3 -c 1 -o gpurun_out/${TAG}_ncu \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu.log
fi
