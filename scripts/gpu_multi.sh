#!/bin/bash
# multi-rank paths on one GPU (ranks share the device; gloo carries the tiny collectives) + the cfg5 sweep at N=1
mkdir -p gpurun_out
TAG=${1:-m}
timeout 900 python bench.py --workload cfg5_2049cubed_f32_chunked_rel1e-4 --steps 3 --warmup 3 > gpurun_out/${TAG}_cfg5_n1.json 2> gpurun_out/${TAG}_cfg5_n1.err
tail -2 gpurun_out/${TAG}_cfg5_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/${TAG}_cfg2_n2.json 2> gpurun_out/${TAG}_cfg2_n2.err
tail -2 gpurun_out/${TAG}_cfg2_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --workload cfg5_2049cubed_f32_chunked_rel1e-4 --steps 2 --warmup 3 > gpurun_out/${TAG}_cfg5_n2.json 2> gpurun_out/${TAG}_cfg5_n2.err
tail -2 gpurun_out/${TAG}_cfg5_n2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
tail -2 gpurun_out/${TAG}_ref.err
