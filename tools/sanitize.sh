#!/bin/bash
# compute-sanitizer memcheck over the small GPU parity cases (one process per test file).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for f in tests/test_gpu_parity.py tests/test_gpu_spadd.py tests/test_gpu_sptrsv.py tests/test_gpu_gcn.py tests/test_gpu_radix.py; do
  b=$(basename $f .py)
  timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
    python -m pytest $f -m gpu -x -q -k "not big and not fullsize and not bench and not huge" > gpurun_out/memcheck_$b.log 2>&1
  echo "$b rc=$? $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/memcheck_$b.log) $(grep 'ERROR SUMMARY' gpurun_out/memcheck_$b.log | tail -1) $(tail -1 gpurun_out/memcheck_$b.log)"
done
