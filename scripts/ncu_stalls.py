"""Summarise an ncu report: key metrics, stall reasons, and per-region stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "launch__registers_per_thread"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
st = [(k, v[i]) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
st = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", "") or 0)) for k, x in st),
            key=lambda t: -t[1])
print("stalls:", ", ".join(f"{k}={int(x)}" for k, x in st if x > 0))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iss]) for r in data)
print("total samples", tot)
marks = ("BAR.SYNC", "LDTM", "SYNCS.PHASECHK", "MUFU.EX2", "EXIT", "USETMAXREG")
acc = 0
last = 0
for n, r in enumerate(data):
    acc += int(r[iss])
    if any(m in r[isrc] for m in marks):
        print(f"{n:5d} {r[isrc][:58]:58s} seg={acc - last:6d} cum={acc}")
        last = acc

# per-region stall reasons: pass regions as a:b pairs after the report path
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for spec in sys.argv[2:]:
    a, b = (int(x) for x in spec.split(":"))
    tot = {c: sum(int(data[n][h.index(c)] or 0) for n in range(a, b)) for c in reasons}
    s = sum(tot.values())
    print(f"region {a}:{b} samples={s}: " + ", ".join(f"{k[6:]}={v}" for k, v in sorted(tot.items(), key=lambda t: -t[1]) if v))
    worst = sorted(range(a, b), key=lambda n: -int(data[n][iss]))[:12]
    for n in sorted(worst):
        top = max(reasons, key=lambda c: int(data[n][h.index(c)] or 0))
        print(f"   {n:5d} {data[n][isrc][:60]:60s} {data[n][iss]:>6s} ({top[6:]})")
