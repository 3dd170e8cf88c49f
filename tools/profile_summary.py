"""Summarise an ncu launch list of `bench.py --steps 1` into per-op device time and DRAM
traffic (cold-cache, serialised replay: compare SHARES, not absolute times).

    python tools/profile_summary.py gpurun_out/launches.csv profiles/r1_ops.json

The launch list must come from
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file <csv> python bench.py --steps 1 --warmup 3 ...
Kernels are attributed to ops by name; the last complete step in the list is used.
"""
from __future__ import annotations

import collections
import csv
import json
import sys

OP_OF = [  # (substring of the kernel name, op) -- order of the step in bench.py
    ("k_col_count", "csr_transpose"), ("k_sort_", "csr_transpose"), ("k_csr_tile<double, 2", "csr_transpose"),
    ("k_rows<double, 2", "csr_transpose"), ("k_rows_long<double, 2", "csr_transpose"),
    ("k_csr_tile<double, 0, 0, 0>", "spmv_fwd"), ("k_csr_tile<double, 0, 1, 1>", "spmv_bwd"),
    ("k_rows<double, 0, 0, 0>", "spmv_fwd"), ("k_rows_long<double, 0, 0, 0>", "spmv_fwd"),
    ("k_rows<double, 1, 0, 1>", "spmv_bwd"), ("k_rows_long<double, 1, 0, 1>", "spmv_bwd"),
    ("k_spmm<double, 8, 4, 0>", "spmm_fwd"), ("k_spmm<double, 8, 4, 3>", "spmm_bwd"),
    ("k_spmm_wide<double, 2, 0", "spmm_fwd"), ("k_spmm_wide<double, 2, 3", "spmm_bwd"),
    ("k_gemm_S<double, 0,", "spgemm_symbolic"), ("k_gemm_W<double, 0,", "spgemm_symbolic"),
    ("k_gemm_big_sym<0,", "spgemm_symbolic"),
    ("k_gemm_S<double, 1,", "spgemm_symbolic"), ("k_gemm_W<double, 1,", "spgemm_symbolic"),
    ("k_gemm_big_sym<1,", "spgemm_symbolic"),
    ("k_gemm_S<double, 2,", "spgemm_numeric"), ("k_gemm_W<double, 2,", "spgemm_numeric"),
    ("k_gemm_big_val<double, 2>", "spgemm_numeric"),
    ("k_gemm_S<double, 3,", "spgemm_bwd"), ("k_gemm_W<double, 3,", "spgemm_bwd"),
    ("k_gemm_big_val<double, 3>", "spgemm_bwd"),
]


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
        k.setdefault(key, {})[r[ci["Metric Name"]]] = float(r[ci["Metric Value"]].replace(",", ""))
    return k


def main(src, dst):
    k = load(src)
    launches = list(k.items())
    # the last step starts at the last transpose column-count kernel
    starts = [i for i, ((_, n), _) in enumerate(launches) if "k_col_count" in n]
    step = launches[starts[-1]:] if starts else launches
    ops = collections.OrderedDict()
    cur = "csr_transpose"  # helper kernels (scans, big-row prep, zero fills) go to the op they sit in
    for (lid, name), m in step:
        op = next((o for s, o in OP_OF if s in name), None)
        if op is None:
            if not name.startswith(("csrk::", "void csrk::")):
                continue
            op = cur
        cur = op
        d = ops.setdefault(op, {"kernels": [], "time_us": 0.0, "dram_bytes": 0.0})
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        d["kernels"].append({"name": name.split("(")[0], "time_us": round(t, 2), "dram_bytes": int(b)})
        d["time_us"] += t
        d["dram_bytes"] += b
    tot = sum(d["time_us"] for d in ops.values())
    for d in ops.values():
        d["share"] = round(d["time_us"] / tot, 4) if tot else None
        d["time_us"] = round(d["time_us"], 2)
        d["dram_bytes"] = int(d["dram_bytes"])
    out = {"source": src, "note": "ncu --clock-control none, serialised cold-cache replay; one bench step",
           "ops": ops}
    json.dump(out, open(dst, "w"), indent=1)
    for o, d in ops.items():
        print(f"{o:18s} {d['time_us']:9.1f} us  share {d['share']:.3f}  dram {d['dram_bytes'] / 1e6:9.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
