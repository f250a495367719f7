"""Per-role (service / S / O warps) dynamic instruction mix and stall breakdown of a
prefill kernel ncu report; roles are delimited by the setmaxnreg instructions."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, tiles = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 33280
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h, data = rows[1], rows[2:]
isrc, iexe = h.index("Source"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
marks = [n for n, r in enumerate(data) if "USETMAXREG" in r[isrc]]
dec = [n for n in marks if "DEALLOC" in data[n][isrc]]
inc = [n for n in marks if "ALLOC" in data[n][isrc] and "DEALLOC" not in data[n][isrc]]
b_s, b_o = dec[-1], inc[0]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"):
    print(f"{k:55s} {rr[2][rr[0].index(k)]}")
for name, (a, z) in {"svc": (0, b_s), "S": (b_s, b_o), "O": (b_o, len(data))}.items():
    c, st, tot = Counter(), Counter(), 0
    for r in data[a:z]:
        try:
            n = int(float(r[iexe] or 0))
        except ValueError:
            n = 0
        op = r[isrc].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += n
        tot += n
        for k in cols:
            try:
                st[k] += int(r[idx[k]] or 0)
            except ValueError:
                pass
    s = sum(st.values()) or 1
    print(f"{name:4s} inst/tile {tot / tiles:7.0f}  samples {s:6d}", [(k, round(v / tiles)) for k, v in c.most_common(12)])
    print("     stalls", {k.replace("stall_", ""): round(v / s, 3) for k, v in st.most_common(9)})
