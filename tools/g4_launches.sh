#!/bin/bash
# per-kernel time + DRAM bytes of one config-4 SpGEMM pass (ncu, serialised) -> gpurun_out/g4_kernels.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g4_launches.csv python tools/gemm4.py --ops ${1:-sym,num,bwd} --reps 1 > gpurun_out/g4_ncu.log 2>&1
python - <<'PY' > gpurun_out/g4_kernels.txt
import csv, collections
rows = list(csv.reader([l for l in open("gpurun_out/g4_launches.csv") if l.startswith('"')]))
h = rows[0]; ci = {x: i for i, x in enumerate(h)}
per = collections.OrderedDict()
for r in rows[1:]:
    k = (r[ci["ID"]], r[ci["Kernel Name"]].split("(")[0][:70])
    d = per.setdefault(k, {})
    d[r[ci["Metric Name"]]] = (float(r[ci["Metric Value"]].replace(",", "")), r[ci["Metric Unit"]])
U = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
for (i, k), d in per.items():
    t = d.get("gpu__time_duration.sum", (0, "us")); t = t[0] * U.get(t[1], 1)
    if t < 200: continue
    b = sum(v[0] * B.get(v[1], 1) for m, v in d.items() if m.startswith("dram"))
    print(f"{i:>5} {k:70s} {t/1e3:9.2f} ms {b/1e9:8.2f} GB")
PY
cat gpurun_out/g4_kernels.txt
