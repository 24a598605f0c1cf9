#!/bin/bash
# launch list (timing only) + one `ncu --set full` pass over every kernel of one bench step; the report is
# summarised on the box (scripts/ncu_all.py) and kept out of gpurun_out (size cap)
mkdir -p gpurun_out /tmp/ncu
TAG=${1:-na}; WL=${2:-cfg2_513cubed_f32_inf_rel1e-4}; SKIP=${3:-160}; CNT=${4:-45}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --launch-skip $SKIP --launch-count $CNT -f -o /tmp/ncu/${TAG}_full \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_full.log 2>&1
python scripts/ncu_all.py /tmp/ncu/${TAG}_full.ncu-rep > gpurun_out/${TAG}_kernels.txt
python scripts/ncu_all.py /tmp/ncu/${TAG}_full.ncu-rep --json > gpurun_out/${TAG}_kernels.json
ls -la /tmp/ncu/
