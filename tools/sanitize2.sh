#!/bin/bash
# compute-sanitizer racecheck / synccheck over a subset of the small GPU parity cases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for tool in racecheck synccheck; do
for f in tests/test_gpu_parity.py tests/test_gpu_sptrsv.py tests/test_gpu_gcn.py tests/test_gpu_spadd.py; do
  b=$(basename $f .py)
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest $f -m gpu -x -q -k "not big and not fullsize and not bench and not huge and not skew" > gpurun_out/${tool}_$b.log 2>&1
  echo "$tool $b rc=$? $(grep -E 'passed|failed' gpurun_out/${tool}_$b.log | tail -1) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/${tool}_$b.log | tail -1)"
done
done
