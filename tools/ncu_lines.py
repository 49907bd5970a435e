"""Aggregate ncu 'cuda,sass' source-page CSV to per-CUDA-line stall samples.
usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
hdr = None
agg = defaultdict(float)
inst = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
src_text = {}
line_key = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] and r[0].isdigit():  # a CUDA source line row
        line_key = (cur_file, int(r[0]))
        src_text[line_key] = r[1][:90]
        continue
    # SASS row under the current CUDA line: columns after the first two
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[line_key] += float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        inst[line_key] += float(d.get("Instructions Executed", 0) or 0)
        for kk, vv in d.items():
            if kk.startswith("stall_") and "Not Issued" not in kk and vv:
                reasons[line_key][kk[6:]] += float(vv)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
top = sorted(agg.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for k, v in top:
    rs = sorted(reasons[k].items(), key=lambda kv: -kv[1])[:3]
    why = " ".join("%s=%.0f%%" % (a, 100 * b / v) for a, b in rs) if v else ""
    print("%6.2f%% %10.0f inst  %s:%d  [%s]  %s" % (100 * v / tot, inst[k], k[0], k[1], why, src_text.get(k, "")[:60]))
