#!/bin/bash
# build, SpGEMM GPU parity tests (-k expr), config-4 SpGEMM op times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/g4tests.log 2>&1; tail -3 gpurun_out/g4tests.log; fi
timeout 900 python tools/gemm4.py --ops ${2:-sym,num,bwd} --reps 3 2>&1 | tail -2
