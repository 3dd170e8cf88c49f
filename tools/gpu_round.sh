#!/bin/bash
# One GPU session: build, the -m gpu suite, the default bench line, and (optionally) the launch
# list + ops trace of the default step attributed to ops (profiles/traffic_cfg2.json source).
#   tools/gpu_round.sh [pytest-args...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; tail -c 300 gpurun_out/bench_default.json
