#!/bin/bash
# A/B the occupancy hint of the GCN propagation (CSRK_GCN_MINB: CTAs of 256 per SM).
cd "$(dirname "$0")/.."
for mb in 1 4 6 8; do
  touch paper_2212_05159_b200/csrc/gcn.cu
  CSRK_NVCC_EXTRA="-DCSRK_GCN_MINB=$mb" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "MINB=$mb $(timeout 600 python bench.py --workload gcn --steps 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: v['ms'] for k, v in d['ops'].items()})")"
done
touch paper_2212_05159_b200/csrc/gcn.cu
