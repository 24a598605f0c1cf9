#!/bin/bash
# full GPU suite, N=1 bench (contract line), launch list of the bench step, reference arm
mkdir -p gpurun_out
TAG=${1:-fin}
(free -g; nproc; lscpu | grep -i 'model name'; nvidia-smi -L) > gpurun_out/${TAG}_host.txt 2>&1
timeout 2400 python -m pytest -m gpu -q -rA --durations=20 tests > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err
tail -1 gpurun_out/${TAG}_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_ncu.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
tail -1 gpurun_out/${TAG}_ref.json | cut -c1-300
