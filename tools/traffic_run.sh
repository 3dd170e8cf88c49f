#!/bin/bash
# ncu launch list (time + DRAM bytes, clocks unlocked) of one bench.py run of workload $1 (extra
# bench args after it) with an --ops-trace of its final pass, then the per-op attribution.
#   tools/traffic_run.sh cfg2        -> gpurun_out/traffic_cfg2.json (copy to profiles/ to commit)
cd "$(dirname "$0")/.."
w=$1; shift
mkdir -p gpurun_out
# CSRK_TRANSPOSE_GRAPH=0: ncu does not replay the kernels of the transpose's conditional graph;
# the stream form launches the same kernels (the general ones gated on the device flag)
CSRK_TRANSPOSE_GRAPH=0 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --print-units base --csv --log-file gpurun_out/launches_$w.csv \
  python bench.py --workload ${w%%_*} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  --ops-trace gpurun_out/trace_$w.json "$@" > gpurun_out/ncu_bench_$w.log 2>&1
echo "ncu rc=$?"
python tools/traffic.py gpurun_out/launches_$w.csv gpurun_out/trace_$w.json gpurun_out/traffic_$w.json
