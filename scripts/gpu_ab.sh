#!/bin/bash
# A/B: parity subset, then the bench phases with the staged fused pass on / off
mkdir -p gpurun_out
TAG=${1:-ab}
timeout 1200 python -m pytest -m gpu -q -x tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -k "not cfg4 and not cfg5" > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
for st in 1 0 1 0; do
  MGRC_FINE_STAGED=$st timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_s$st.json 2>> gpurun_out/${TAG}_bench.err
  TAG=${TAG} ST=$st python - <<"PY"
import json,os
d=json.loads(open(f"gpurun_out/{os.environ['TAG']}_bench_s{os.environ['ST']}.json").read().strip().splitlines()[-1])
print("staged", os.environ['ST'], round(d["value"],1), "c", round(d["compress_gbs"],1), "d", round(d["decompress_gbs"],1), {k:v["ms"] for k,v in list(d["phases_ms_per_step"].items())[:5]})
PY
done
timeout 300 python scripts/tfd_probe.py > gpurun_out/${TAG}_tfd_probe.log 2>&1; tail -5 gpurun_out/${TAG}_tfd_probe.log
