#!/bin/bash
# A/B of the e2e number (pipelined H2D / step / D2H) under the launch / cache knobs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for env in "X=1" "CSRK_PDL=0" "CSRK_GEMM_FILL_CACHE=0" "X=1"; do
  env $env timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/ab_e2e.log 2>&1
  tail -1 gpurun_out/ab_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done
