#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the container, decoder, chunked and MDR tests
mkdir -p gpurun_out
TAG=${1:-san}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "container_parity and (33x17x9 or 257x256) or corrupt or chunked_parity" \
    > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/${TAG}_summary.txt
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_mdr.py -k "33x17x9 or 17-B8" \
    > gpurun_out/${TAG}_${tool}_mdr.log 2>&1
  echo "$tool mdr rc=$?" | tee -a gpurun_out/${TAG}_summary.txt
done
