#!/bin/bash
# ncu --set full of the config-2 SpMM kernels: forward (mode 0) and fused backward (mode 3), one launch each.
#   tools/ncu_spmm.sh [suffix]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for md in 0 3; do
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_spmm_pipe<double, \\(int\\)2, \\(int\\)$md" -c 1 -o gpurun_out/full_spmm$md${1:-} python tools/micro.py --ops spmm --reps 1 > gpurun_out/ncu_spmm$md.log 2>&1
  python tools/ncu_summary.py gpurun_out/full_spmm$md${1:-}.ncu-rep gpurun_out/full_spmm$md${1:-}.txt
  ncu -i gpurun_out/full_spmm$md${1:-}.ncu-rep --page raw --csv > gpurun_out/full_spmm$md${1:-}_raw.csv 2>/dev/null
  ncu -i gpurun_out/full_spmm$md${1:-}.ncu-rep --page source --csv > gpurun_out/full_spmm$md${1:-}_src.csv 2>/dev/null
done
