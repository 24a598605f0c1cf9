#!/bin/bash
# Round-2 bench contract check: N=1 default, N=2 (self-launched; shared GPU -> gloo), reference arm.
mkdir -p gpurun_out
TAG=${1:-b}
(free -g; nproc; lscpu | grep -i 'model name'; nvidia-smi -L) > gpurun_out/${TAG}_host.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err
tail -2 gpurun_out/${TAG}_n1.err
timeout 1200 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/${TAG}_n2.json 2> gpurun_out/${TAG}_n2.err
tail -2 gpurun_out/${TAG}_n2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
tail -2 gpurun_out/${TAG}_ref.err
