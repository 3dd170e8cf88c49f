#!/bin/bash
# GPU-box check used during development: build, GPU tests (optional filter), benches.
#   tools/gpu_check.sh "<pytest -k expr or empty>" "<bench workloads, e.g. cfg2 cfg4>"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then
  if [ "$1" = "all" ]; then
    timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
  else
    timeout 1500 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/gputests.log 2>&1
  fi
  tail -3 gpurun_out/gputests.log
fi
for w in $2; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.log 2>&1
  tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['ops'].items()})" 2>&1 | tail -2
done
