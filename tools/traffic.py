"""Attribute an ncu launch list of a bench.py run to the ops of its --ops-trace pass.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/L.csv \
        python bench.py --workload W --steps 1 --warmup 3 --ops-trace gpurun_out/T.json ...
    python tools/traffic.py gpurun_out/L.csv gpurun_out/T.json profiles/traffic_W.json

The trace lists, in launch order, how many csrk kernels each op of the final pass launched; the
last sum(counts) csrk kernels of the launch list are that pass.  Output per op: device time and
DRAM bytes (read + write) summed over its kernels -- cold-cache serialised replay, so compare
shares and bytes, not absolute times.  bench.py reads the bytes as roofline.traffic.
"""
from __future__ import annotations

import collections
import csv
import json
import sys


UNIT = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "byte": 1.0,
        "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}   # -> ns and bytes


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ci = {h: i for i, h in enumerate(hdr)}
    k = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[ci["ID"]]), r[ci["Kernel Name"]])
        scale = UNIT.get(r[ci["Metric Unit"]].strip().lower(), 1.0) if "Metric Unit" in ci else 1.0
        k.setdefault(key, {})[r[ci["Metric Name"]]] = float(r[ci["Metric Value"]].replace(",", "")) * scale
    return [(name, m) for (_, name), m in sorted(k.items(), key=lambda kv: kv[0][0])]


def is_csrk(name):
    """A csrk kernel: namespaced (stream launches) or, for CUDA-graph kernel nodes (which ncu names
    without the namespace), a k_* function that is not a torch / library kernel."""
    if "csrk::" in name:
        return True
    head = name.strip()
    if head.startswith("void "):
        head = head[5:]
    head = head.split("(")[0].split("<")[0].strip()
    return head.startswith("k_") and "::" not in head


def main(csv_path, trace_path, out_path):
    kern = [(n, m) for n, m in load(csv_path) if is_csrk(n)]
    trace = json.load(open(trace_path))["ops"]
    total = sum(c for _, c in trace)
    if total > len(kern):
        raise SystemExit(f"trace has {total} launches, launch list only {len(kern)} csrk kernels")
    kern = kern[len(kern) - total:]
    ops, i = {}, 0
    for op, cnt in trace:
        ks = kern[i:i + cnt]
        i += cnt
        ent = ops.setdefault(op, {"time_us": 0.0, "dram_bytes": 0, "kernels": []})
        for name, m in ks:
            t = m.get("gpu__time_duration.sum", 0.0)      # ns
            b = int(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
            ent["time_us"] += t / 1000.0
            ent["dram_bytes"] += b
            ent["kernels"].append({"name": name.split("(")[0], "time_us": round(t / 1000.0, 2), "dram_bytes": b})
        ent["time_us"] = round(ent["time_us"], 2)
    json.dump({"source": csv_path, "trace": trace_path,
               "note": "ncu --clock-control none, serialised cold-cache replay; the final --ops-trace pass",
               "ops": ops}, open(out_path, "w"), indent=1)
    print(json.dumps({k: (v["time_us"], v["dram_bytes"]) for k, v in ops.items()}))


if __name__ == "__main__":
    main(*sys.argv[1:4])
