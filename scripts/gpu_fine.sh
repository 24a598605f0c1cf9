#!/bin/bash
# fused-pass iteration: parity subset, bench phases (x2), optional ncu capture of $NCU_K
mkdir -p gpurun_out
TAG=${1:-f}
timeout 1200 python -m pytest -m gpu -q -x tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_l2proj.py -k "not cfg4 and not cfg5" > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b$i.json 2>> gpurun_out/${TAG}_bench.err
  F=gpurun_out/${TAG}_b$i.json python - <<"PY"
import json,os
d=json.loads(open(os.environ["F"]).read().strip().splitlines()[-1])
p=d["phases_ms_per_step"]
print(round(d["value"],1), "c", round(d["compress_gbs"],1), "d", round(d["decompress_gbs"],1), {k:v["ms"] for k,v in list(p.items())[:6]})
PY
done
if [ -n "$NCU_K" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_K} -s 3 -c 1 -o gpurun_out/${TAG}_ncu \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
  tail -1 gpurun_out/${TAG}_ncu.log
fi
