"""Dynamic opcode histogram of an ncu report's SASS source page per work unit:
    python scripts/ncu_ophist.py <report.ncu-rep> <units (e.g. tiles or pages)>"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]; units = float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[start]; isrc = h.index("Source"); iex = h.index("Instructions Executed")
c = Counter()
for r in rows[start+1:]:
    if len(r) < len(h): continue
    s = r[isrc].strip()
    if not s: continue
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    c[op.split(".")[0]] += int(r[iex] or 0)
tot = sum(c.values())
print("total per unit", tot/units)
for k, v in c.most_common(30): print(f"{k:12s} {v/units:8.1f}")
