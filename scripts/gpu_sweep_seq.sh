#!/bin/bash
# subsequence length x warm-up sweep of the decoder (cfg2 phases); parity checked per build
mkdir -p gpurun_out
for SB in ${SEQS:-512 1024}; do for W in ${WARMS:-256 512}; do
  MGRC_NVCC_EXTRA="-DMGRC_WARM_BITS=$W -DMGRC_SEQ_BITS=$SB" python paper_2401_05994_b200/build.py --force > /dev/null 2>&1 || { echo "build $SB/$W failed"; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "container_parity or slab" > gpurun_out/seq_${SB}_${W}_pytest.log 2>&1; tail -1 gpurun_out/seq_${SB}_${W}_pytest.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/seq_${SB}_$W.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/seq_${SB}_$W.json')); p=d['phases_ms_per_step']
print($SB, $W, round(d['value'],1), round(d['decompress_gbs'],1), {k: v['ms'] for k, v in p.items() if k.startswith('huff')})"
done; done
