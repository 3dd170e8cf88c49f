#!/bin/bash
# ncu launch list (duration + DRAM bytes) of one micro.py op group: tools/launches.sh <ops> [extra env]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
env $2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launch_$1.csv python tools/micro.py --ops $1 --reps 1 > /dev/null 2>&1
python - "$1" <<'PY'
import csv, sys
rows = list(csv.reader([l for l in open(f"gpurun_out/launch_{sys.argv[1]}.csv") if l.startswith('"')]))
h = rows[0]; ci = {x: i for i, x in enumerate(h)}
k = {}
order = []
for r in rows[1:]:
    if len(r) < len(h): continue
    key = (int(r[ci["ID"]]), r[ci["Kernel Name"]][:70], r[ci["Grid Size"]])
    if key not in k: k[key] = {}; order.append(key)
    k[key][r[ci["Metric Name"]]] = r[ci["Metric Value"]]
for key in order[-40:]:
    m = k[key]
    print(f"{key[0]:4d} {key[1]:70s} {key[2]:>14s} {float(m.get('gpu__time_duration.sum', 0))/1e3:8.2f} us "
          f"{(float(m.get('dram__bytes_read.sum', 0)) + float(m.get('dram__bytes_write.sum', 0)))/1e6:8.1f} MB")
PY
