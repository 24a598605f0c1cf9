#!/bin/bash
# GPU test suite with per-test durations; args: TAG [pytest selectors...]
mkdir -p gpurun_out
TAG=${1:-t}; shift
timeout 3000 python -m pytest -m gpu -q -rA --durations=30 "${@:-tests}" > gpurun_out/${TAG}_pytest.log 2>&1
tail -40 gpurun_out/${TAG}_pytest.log
