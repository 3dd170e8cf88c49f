#!/bin/bash
# Default bench line + the --set full capture only (see refresh_profiles.sh).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 1200 ncu -f --set full --import-source on --clock-control none \
  -k 'regex:k_spmm_wide|k_gemm_S|k_sort_short|k_col_count|k_rows' -c 22 \
  -o gpurun_out/full_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -c 300 gpurun_out/bench_default.log
