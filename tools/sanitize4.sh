#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for tool in memcheck racecheck; do
for f in tests/test_gpu_radix.py tests/test_gpu_validate.py tests/test_pcg.py tests/test_spai.py; do
  b=$(basename $f .py)
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest $f -m gpu -x -q -k "not config5 and not slow and not fullsize" > gpurun_out/${tool}_$b.log 2>&1
  echo "${tool}_$b: $(grep -E 'passed|failed' gpurun_out/${tool}_$b.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${tool}_$b.log | tail -1 | sed 's/=========//')"
done
done
