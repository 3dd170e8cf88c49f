#!/bin/bash
# Per-kernel time breakdown of one config-5 PCG step (ncu, duration only, serialised) -> gpurun_out/cfg5_kernels.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
CSRK_PCG_GRAPH=0 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/cfg5_launches.csv python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/cfg5_ncu.log 2>&1
python - <<'PY' > gpurun_out/cfg5_kernels.txt
import csv, collections
rows = list(csv.reader([l for l in open("gpurun_out/cfg5_launches.csv") if l.startswith('"')]))
h = rows[0]; ci = {x: i for i, x in enumerate(h)}
per = collections.defaultdict(lambda: [0.0, 0.0, set()])
for r in rows[1:]:
    k = r[ci["Kernel Name"]].split("(")[0][:60]
    m, v, u = r[ci["Metric Name"]], float(r[ci["Metric Value"]].replace(",", "")), r[ci["Metric Unit"]]
    scale = {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(u, 1)
    if m == "gpu__time_duration.sum": per[k][0] += v * scale; per[k][2].add(r[ci["ID"]])
    elif m.startswith("dram__bytes"):
        per[k][1] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
tot = sum(v[0] for v in per.values())
print(f"total {tot/1e3:.1f} ms over {sum(len(v[2]) for v in per.values())} launches")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:60s} {v[0]/1e3:9.2f} ms {100*v[0]/tot:5.1f}%  {v[1]/1e9:8.2f} GB  launches {len(v[2])}")
PY
cat gpurun_out/cfg5_kernels.txt
