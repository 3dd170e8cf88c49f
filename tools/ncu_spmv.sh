#!/bin/bash
# ncu --set full of the config-2 SpMV kernels (forward REDUCE, backward SCATTER+SIDE), CSRK_SPMV_SLOT=$1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
export CSRK_SPMV_SLOT=${1:-1}
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_rows<double, \\(int\\)1, \\(bool\\)0, \\(bool\\)1>" -c 1 -o gpurun_out/full_spmv$1 python tools/micro.py --ops spmv --reps 1 > gpurun_out/ncu_spmv.log 2>&1
python tools/ncu_summary.py gpurun_out/full_spmv$1.ncu-rep gpurun_out/full_spmv$1.txt
ncu -i gpurun_out/full_spmv$1.ncu-rep --page raw --csv > gpurun_out/full_spmv$1_raw.csv 2>/dev/null
