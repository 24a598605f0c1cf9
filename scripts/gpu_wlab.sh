#!/bin/bash
# A/B of build variants ($VARIANTS) on bench workloads ($WLS): round-trip GB/s and the fine phase
for v in ${VARIANTS}; do
  f="${v//,/ }"
  MGRC_NVCC_EXTRA="$f" timeout 900 python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || { echo "build $f failed"; continue; }
  for wl in ${WLS}; do
    timeout 900 python bench.py --workload $wl --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e > /tmp/wl.json 2>/tmp/wl.err
    V="$f" WL=$wl python - <<"PY"
import json,os
try:
    d=json.loads(open("/tmp/wl.json").read().strip().splitlines()[-1])
    p=d.get("phases_ms_per_step",{})
    print(os.environ["V"], os.environ["WL"], round(d["value"],1), {k:v["ms"] for k,v in list(p.items())[:4]})
except Exception as e:
    print(os.environ["V"], os.environ["WL"], "ERR", open("/tmp/wl.err").read()[-300:])
PY
  done
done
