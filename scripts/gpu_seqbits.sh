#!/bin/bash
# subsequence-length sweep of the Huffman decoder (cfg2 + a cfg5 slab)
mkdir -p gpurun_out
TAG=${1:-sq}
for v in ${VARIANTS:-"-DMGRC_SEQ_BITS=1024" "-DMGRC_SEQ_BITS=2048" "-DMGRC_SEQ_BITS=4096"}; do
  MGRC_NVCC_EXTRA="$v" timeout 900 python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/${TAG}_build.log 2>&1 || { echo "build $v failed"; tail -5 gpurun_out/${TAG}_build.log; continue; }
  echo "$v"
  timeout 600 python scripts/tfd_probe.py 2>&1 | tail -2
done
