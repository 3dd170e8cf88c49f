#!/bin/bash
# Round profile refresh: launch list of one default bench step (ncu, time + DRAM bytes), the
# default bench line, and every workload's bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_bench.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
for w in cfg3 cfg4 cfg5 trsv gcn f12; do
  timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.log 2>&1
done
timeout 900 python bench.py --workload cfg5 --precond solve --steps 5 > gpurun_out/bench_cfg5_solve.log 2>&1
# one --set full capture of the main kernels: the workload set-up (plan, symbolic) + the first warm-up step
timeout 1200 ncu -f --set full --import-source on --clock-control none \
  -k 'regex:k_spmm_pipe|k_gemm_S|k_tr_sym|k_rows' -c 16 \
  -o gpurun_out/full_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -c 400 gpurun_out/bench_default.log
# per-op attribution of the default step (profiles/traffic_cfg2.json source)
bash tools/traffic_run.sh cfg2 > gpurun_out/traffic_run.log 2>&1
