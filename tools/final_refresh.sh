#!/bin/bash
# Round-end evidence refresh (one GPU call): per-workload ncu launch lists attributed to ops
# (profiles/traffic_<w>.json, read by bench.py for roofline.traffic), then every bench line, then
# a --set full capture of the default step's main kernels.  Outputs under gpurun_out/final/.
cd "$(dirname "$0")/.."
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for w in cfg2 cfg3 cfg4 cfg5 trsv gcn f12; do
  bash tools/traffic_run.sh $w > $O/traffic_run_$w.log 2>&1
  cp gpurun_out/traffic_$w.json profiles/traffic_$w.json 2>/dev/null && cp gpurun_out/traffic_$w.json $O/
  cp gpurun_out/launches_$w.csv $O/ 2>/dev/null
  echo "traffic $w: $(tail -1 $O/traffic_run_$w.log)"
done
timeout 900 python bench.py > $O/bench_line.json 2> $O/bench_default.err; echo "bench rc=$?"
for w in cfg3 cfg4 cfg5 trsv gcn f12; do
  timeout 900 python bench.py --workload $w --steps 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"
done
timeout 900 python bench.py --workload cfg5 --precond solve --steps 5 > $O/bench_cfg5_solve.json 2> $O/bench_cfg5_solve.err
timeout 1200 ncu -f --set full --import-source on --clock-control none \
  -k 'regex:k_spmm_pipe|k_gemm_S|k_tr_sym|k_rows' -c 16 \
  -o $O/full_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -c 600 $O/bench_line.json
