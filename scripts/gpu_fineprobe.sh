#!/bin/bash
# fused-pass diagnostic builds ($VARIANTS, comma = space inside one variant), fine-phase ms each
for v in ${VARIANTS}; do
  f="${v//,/ }"
  MGRC_NVCC_EXTRA="$f" timeout 900 python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || { echo "build $f failed"; continue; }
  timeout 300 python scripts/fine_probe.py "$f" 2>&1 | tail -1
done
