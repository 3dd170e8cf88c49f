#!/bin/bash
# ncu --set full of the symbolic COUNT and FILL short-row kernels on config 2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for ph in 0 1; do
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_gemm_S<double, \\(int\\)$ph" -c 1 -o gpurun_out/full_sym$ph python tools/micro.py --ops gemm --reps 1 > gpurun_out/ncu_sym.log 2>&1
python tools/ncu_summary.py gpurun_out/full_sym$ph.ncu-rep gpurun_out/full_sym$ph.txt
ncu -i gpurun_out/full_sym$ph.ncu-rep --page raw --csv > gpurun_out/full_sym${ph}_raw.csv 2>/dev/null
ncu -i gpurun_out/full_sym$ph.ncu-rep --page source --csv > gpurun_out/full_sym${ph}_src.csv 2>/dev/null
done
