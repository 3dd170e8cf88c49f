#!/bin/bash
# A/B: programmatic dependent launch on/off over the bench workloads (steps 10).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for w in ${WL:-cfg2 trsv gcn cfg5}; do
  for pdl in 1 0 1 0; do
    CSRK_PDL=$pdl timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/ab_pdl_$w.log 2>&1
    tail -1 gpurun_out/ab_pdl_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w pdl=$pdl', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['ops'].items()})" 2>&1 | tail -1
  done
done
