#!/bin/bash
# decoder bring-up: parity subset (incl. byte-flip fuzz), then bench phases (new and old decoder), cfg5 slab decode
mkdir -p gpurun_out
TAG=${1:-d}
timeout 1200 python -m pytest -m gpu -q -x tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -k "not cfg4 and not cfg5" > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err

timeout 900 python bench.py --workload cfg5_2049cubed_f32_chunked_rel1e-4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
TAG=${TAG} python - <<"PY"
import json,sys
for f in ["bench","cfg5"]:
    try:
        d=json.loads(open(f"gpurun_out/{__import__('os').environ['TAG']}_{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"],1), "c", round(d["compress_gbs"],1), "d", round(d["decompress_gbs"],1), {k:v["ms"] for k,v in list(d.get("phases_ms_per_step", d.get("phases_ms_per_step_rank0",{})).items())[:6]})
    except Exception as e: print(f, "ERR", e)
PY
