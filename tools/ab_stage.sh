#!/bin/bash
# A/B: SpGEMM shared-memory staging knobs (FILL / NUM+BWD) on config 2 and 3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for w in cfg2 cfg3; do
  for env in "X=1" "CSRK_GEMM_STAGE_FILL=0" "CSRK_GEMM_STAGE_VALS=1" "X=1"; do
    env $env timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_stage.log 2>&1
    tail -1 gpurun_out/ab_stage.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $env', d['ms_per_step'], {k: v['ms'] for k, v in d['ops'].items() if 'spgemm' in k})"
  done
done
