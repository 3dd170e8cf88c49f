#!/bin/bash
# A/B the plan-path SpMV backward split (CSRK_SPMV_PLAN_SPLIT) on config 2 (micro) and config 4 (bench).
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in 0 1; do
  echo "split=$v cfg2 $(CSRK_SPMV_PLAN_SPLIT=$v python tools/micro.py --ops spmv --reps 20 | cut -c1-80)"
  CSRK_SPMV_PLAN_SPLIT=$v timeout 600 python bench.py --workload cfg4 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$v cfg4', {k: v['ms'] for k, v in d['ops'].items() if 'spmv' in k})"
done
