#!/bin/bash
# bench lines of the extra workloads (J1 transform round trip, f3 correction)
mkdir -p gpurun_out
TAG=${1:-w}
for wl in cfg4_1025cubed_f64_roundtrip cfg4_1025cubed_f64_roundtrip_l2proj cfg2_513cubed_f32_inf_rel1e-4_l2proj; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$wl.json 2> gpurun_out/${TAG}_$wl.err
  tail -c 600 gpurun_out/${TAG}_$wl.json; echo; tail -2 gpurun_out/${TAG}_$wl.err
done
