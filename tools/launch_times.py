"""Device time of each launch of one cfg4 batch solve (probe / order / main /
finish), read from an ncu launch list: python tools/launch_times.py <csv>..."""
import csv
import sys

for path in sys.argv[1:]:
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"][:60], r["Block Size"], float(r["Metric Value"].replace(",", ""))))
    print(path)
    for k, b, v in rows:
        unit = 1e-6 if v > 1e5 else 1e-3
        print(f"  {k:60s} {b:>14s} {v / 1e6:10.3f} ms")
