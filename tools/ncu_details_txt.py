"""ncu --page details --csv -> 'Section | Metric | Value Unit' lines (the
format of profiles/*_details.txt): python tools/ncu_details_txt.py in.csv [kernel-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = {k: i for i, k in enumerate(rows[0])}
pat = sys.argv[2] if len(sys.argv) > 2 else ""
kernel = None
for r in rows[1:]:
    if len(r) <= h["Metric Value"] or not r[h["Metric Name"]] or pat not in r[h["Kernel Name"]]:
        continue
    kernel = r[h["Kernel Name"]]
    unit = r[h["Metric Unit"]]
    print(f'{r[h["Section Name"]]} | {r[h["Metric Name"]]} | {r[h["Metric Value"]]} {unit}'.rstrip())
if kernel:
    print(f"Kernel: {kernel} Block {r[h['Block Size']]} Grid {r[h['Grid Size']]}")
