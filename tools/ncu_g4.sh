#!/bin/bash
# --set full capture of the config-4 numeric kernels (W warp path + big-row windows):
#   tools/ncu_g4.sh [ops] [kernel regex]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
OPS=${1:-num}
RE=${2:-'regex:k_gemm_W<float, \(int\)2|k_gemm_big_win<float, \(int\)2'}
timeout 600 python tools/gemm4.py --ops $OPS --reps 3 > gpurun_out/g4_plain.json 2>&1; tail -2 gpurun_out/g4_plain.json
timeout 1500 ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k "$RE" -c 2 \
  -o gpurun_out/full_g4 python tools/gemm4.py --ops $OPS --reps 1 > gpurun_out/ncu_g4.log 2>&1
tail -c 300 gpurun_out/ncu_g4.log
