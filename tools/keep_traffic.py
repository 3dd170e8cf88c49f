"""Copy a gpurun_out traffic capture into profiles/ (committed): the launch list, the ops trace and
the attribution, with the attribution's `source` pointing at the committed copies.

    python tools/keep_traffic.py cfg2 r2      -> profiles/r2_launches_cfg2.csv, profiles/traffic_cfg2.json
"""
import json
import shutil
import sys

w, tag = sys.argv[1], sys.argv[2]
csv_dst = f"profiles/{tag}_launches_{w}.csv"
tr_dst = f"profiles/{tag}_trace_{w}.json"
shutil.copy(f"gpurun_out/launches_{w}.csv", csv_dst)
shutil.copy(f"gpurun_out/trace_{w}.json", tr_dst)
d = json.load(open(f"gpurun_out/traffic_{w}.json"))
d["source"], d["trace"] = csv_dst, tr_dst
json.dump(d, open(f"profiles/traffic_{w}.json", "w"), indent=1)
print({k: (v["time_us"], v["dram_bytes"]) for k, v in d["ops"].items()})
