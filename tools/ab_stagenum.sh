#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "spgemm or spai or fullsize" > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log
for w in cfg3 cfg2 cfg4; do
  for env in "X=1" "CSRK_GEMM_STAGE_NUM=0"; do
    env $env timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_sn.log 2>&1
    tail -1 gpurun_out/ab_sn.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $env', d['ms_per_step'], {k: v['ms'] for k, v in d['ops'].items() if 'numeric' in k})"
  done
done
