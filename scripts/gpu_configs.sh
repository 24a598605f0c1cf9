#!/bin/bash
# every BASELINE.json config through bench.py (one line each) + compute-sanitizer memcheck on small parity cases
mkdir -p gpurun_out
TAG=${1:-c}
for W in cfg1_65cubed_f64_inf_rel1e-3 cfg2_513cubed_f32_inf_rel1e-4 cfg3_8193sq_f64_s1_rel1e-3 cfg4_1025cubed_f64_inf_rel1e-5; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_$W.json 2> gpurun_out/${TAG}_$W.err
done
timeout 900 python bench.py --workload cfg5_2049cubed_f32_chunked_rel1e-4 --steps 2 --warmup 3 > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "container_parity and (65x65x65 or 33x17x9 or 129x130 or 6x5x4x3 or 17-) or chunked or constant or error_paths" \
  > gpurun_out/${TAG}_memcheck.log 2>&1
tail -5 gpurun_out/${TAG}_memcheck.log
