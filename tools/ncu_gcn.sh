#!/bin/bash
# ncu --set full of the GCN propagation kernels (forward and backward, one launch each).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_gcn_prop<|k_gcn_deg" -c 3 -o gpurun_out/full_gcn${1:-} python bench.py --workload gcn --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gcn.log 2>&1
python tools/ncu_summary.py gpurun_out/full_gcn${1:-}.ncu-rep gpurun_out/full_gcn${1:-}.txt
ncu -i gpurun_out/full_gcn${1:-}.ncu-rep --page raw --csv > gpurun_out/full_gcn${1:-}_raw.csv 2>/dev/null
