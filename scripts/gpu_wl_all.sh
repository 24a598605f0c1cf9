#!/bin/bash
# refresh the non-default bench lines: N=2 chunked (configs[4], ranks sharing the GPU), cfg4 round trip,
# cfg4 container workload, cfg3, cfg2 with the L2 projection
mkdir -p gpurun_out
TAG=${1:-wl}
timeout 1500 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/${TAG}_n2.json 2> gpurun_out/${TAG}_n2.err; tail -1 gpurun_out/${TAG}_n2.err
for wl in cfg4_1025cubed_f64_roundtrip cfg4_1025cubed_f64_inf_rel1e-5 cfg3_8193sq_f64_s1_rel1e-3 cfg2_513cubed_f32_inf_rel1e-4_l2proj; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/${TAG}_$wl.json 2> gpurun_out/${TAG}_$wl.err; tail -1 gpurun_out/${TAG}_$wl.err
done
for f in gpurun_out/${TAG}_*.json; do python - "$f" <<"PY"
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"],1), d.get("compress_gbs"), d.get("decompress_gbs"), (d.get("e2e") or {}).get("value"))
PY
done
