#!/bin/bash
# config-4 SpGEMM op times under build variants: tools/ab_g4.sh ops "<nvcc extra flags>" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ops=$1; shift
for v in "$@"; do
  CSRK_NVCC_EXTRA="$v" python -c "from paper_2212_05159_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1 || tail -5 gpurun_out/b.log
  echo "[$v] $(timeout 900 python tools/gemm4.py --ops $ops --reps 3 2>&1 | tail -1)"
done
