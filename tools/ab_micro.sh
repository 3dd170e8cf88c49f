#!/bin/bash
# config-2 micro-benchmark under build variants: tools/ab_micro.sh ops "<nvcc extra flags>" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ops=$1; shift
for v in "$@"; do
  CSRK_NVCC_EXTRA="$v" python -c "from paper_2212_05159_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1 || tail -5 gpurun_out/b.log
  echo "[$v] $(timeout 900 python tools/micro.py --ops $ops --reps 20 2>&1 | tail -1)"
done
