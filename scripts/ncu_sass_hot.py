#!/usr/bin/env python3
"""Per-instruction view of an ncu report's source page (SASS): executed warp-instructions
and stall samples, bucketed into address windows, plus the top stalled instructions.
    python scripts/ncu_sass_hot.py <report.ncu-rep> [bucket_instrs=64] [kernel_regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[start]
ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [(i, k[len("stall_"):]) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
data, rs = [], []
for r in rows[start + 1:]:
    if len(r) < len(h) or not r[ia].startswith("0x"):
        continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)))
    rs.append({k: int(r[i] or 0) for i, k in reasons})
base = data[0][0]
tot_s = sum(d[2] for d in data); tot_e = sum(d[3] for d in data)
print(f"instructions executed {tot_e}, stall samples {tot_s}")
for i in range(0, len(data), bucket):
    chunk = data[i:i + bucket]
    s = sum(d[2] for d in chunk); e = sum(d[3] for d in chunk)
    if s or e:
        ops = {}
        for d in chunk:
            op = d[1].split()[0] if not d[1].startswith("@") else d[1].split()[1]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + d[3]
        top = sorted(ops.items(), key=lambda x: -x[1])[:4]
        rr = {}
        for d in rs[i:i + bucket]:
            for k, v in d.items():
                rr[k] = rr.get(k, 0) + v
        rtop = " ".join(f"{k}:{v}" for k, v in sorted(rr.items(), key=lambda x: -x[1])[:4] if v)
        print(f"[{i:5d}-{i+len(chunk)-1:5d}] exec {e:10d} ({100*e/tot_e:5.1f}%) stalls {s:7d} ({100*s/tot_s:5.1f}%)  {top}\n      {rtop}")
tot = {}
for d in rs:
    for k, v in d.items():
        tot[k] = tot.get(k, 0) + v
print("stall reasons:", " ".join(f"{k}:{v}" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
print("top stalled instructions:")
for d in sorted(data, key=lambda x: -x[2])[:25]:
    print(f"  {(d[0]-base)//16:5d} {d[2]:6d} {d[3]:9d}  {d[1][:80]}")
