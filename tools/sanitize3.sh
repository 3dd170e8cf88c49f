#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spgemm and not big" > gpurun_out/racecheck_spgemm.log 2>&1
grep -E 'passed|failed|RACECHECK SUMMARY' gpurun_out/racecheck_spgemm.log | tail -2
grep -o "in spgemm.cu:[0-9]*" gpurun_out/racecheck_spgemm.log | sort | uniq -c | head
for w in cfg4; do
  timeout 600 python bench.py --workload $w --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$w.log 2>&1
  tail -1 gpurun_out/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], {k: v['ms'] for k, v in d['ops'].items() if 'spgemm' in k})"
done
