#!/bin/bash
# A/B: SpGEMM symbolic FILL from the COUNT-phase column cache vs a second merge.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "spgemm or spai or symbolic" > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
for w in ${WL:-cfg2 cfg3 cfg2}; do
  for c in 1 0; do
    CSRK_GEMM_FILL_CACHE=$c timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_fc_$w.log 2>&1
    tail -1 gpurun_out/ab_fc_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w cache=$c', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['ops'].items() if 'spgemm' in k})" 2>&1 | tail -1
  done
done
