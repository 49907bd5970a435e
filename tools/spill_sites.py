"""Local-memory (spill) instruction sites of one kernel, by innermost source
line: python tools/spill_sites.py <object.o> <kernel-name-substring>.
Runs cuobjdump -xelf + nvdisasm -gi (line info with inlining)."""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
fn, cur, prev_instr = None, None, True
cnt = collections.Counter()
for l in sass.splitlines():
    if l.startswith(".text."):
        fn = l[6:].rstrip(":")
        continue
    if not fn or pat not in fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if prev_instr:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        prev_instr = False
        continue
    if re.search(r"/\*[0-9a-f]+\*/", l):
        prev_instr = True
        if re.search(r"\b(STL|LDL)(\.\w+)?\b", l):
            cnt[cur] += 1
for k, v in cnt.most_common(60):
    print(f"{v:5d}  {k}")
print("total", sum(cnt.values()))
