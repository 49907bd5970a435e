"""DRAM traffic of one cfg4 bench step from ONE ncu session over every launch
of the step (probe, order, main, finish): writes profiles/traffic.json, read
by bench.py for roofline.traffic.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/one_batch.py
  python tools/traffic.py gpurun_out/traffic.csv [profiles/traffic.json]
"""
import csv
import json
import sys
from collections import OrderedDict

src = sys.argv[1]
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
with open(src) as f:
    lines = [l for l in f if l.startswith('"')]
launches = OrderedDict()
for r in csv.DictReader(lines):
    key = (r["ID"], r["Kernel Name"])
    d = launches.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0], "block": r["Block Size"],
                                  "grid": r["Grid Size"]})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    if r["Metric Name"].startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r["Metric Name"]] = v
    elif r["Metric Name"] == "gpu__time_duration.sum":
        d["ms"] = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
rows = list(launches.values())
solve = [d for d in rows if "solve" in d["kernel"]]
step = [d for d in rows if "pack" not in d["kernel"]]
tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in step)
out = {"source": "one ncu session (--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none) over every launch of one cfg4 batch solve (tools/one_batch.py)",
       "launches": rows, "dram_bytes_per_step": tot,
       "dram_bytes_per_launch": tot,  # bench.py's roofline treats the step as one launch sequence
       "device_ms_per_step_under_ncu": sum(d.get("ms", 0) for d in step)}
json.dump(out, open(dst, "w"), indent=1)
for d in rows:
    print(f"{d['kernel'][:50]:50s} {d['block']:>12s} {d.get('ms', 0):9.3f} ms "
          f"read {d.get('dram__bytes_read.sum', 0) / 1e9:7.2f} GB write {d.get('dram__bytes_write.sum', 0) / 1e9:7.2f} GB")
print(f"step DRAM {tot / 1e9:.1f} GB -> {dst}")
