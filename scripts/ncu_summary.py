#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py <tag>        # reads gpurun_out/<tag>_{launches.csv,prefill,decode}.ncu-rep

Writes profiles/<tag>.md (launch shares + key metrics per captured kernel) and
merges DRAM traffic per launch into profiles/ncu_traffic.json (bench.py's
roofline "traffic" field).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def raw_page(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def summarise_rep(rep):
    lines = []
    kernels = raw_page(rep)
    res = []
    for k in kernels:
        name = k.get("Kernel Name", ("?", ""))[0]
        lines.append(f"### `{name[:160]}`\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for key in KEYS:
            if key in k:
                lines.append(f"| {key} | {k[key][0]} | {k[key][1]} |")
        stalls = sorted(((float(v[0].replace(",", "") or 0), n[len(STALL_PREFIX):]) for n, v in k.items()
                         if n.startswith(STALL_PREFIX) and n.endswith(".ratio")
                         and v[0].replace(",", "").replace(".", "").isdigit()), reverse=True)[:6]
        if stalls:
            lines.append("\nTop warp stall reasons (cycles per issued instruction): " +
                         ", ".join(f"{n.replace('.ratio', '')} {v:.2f}" for v, n in stalls))
        rd = to_bytes(*k["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in k else None
        wr = to_bytes(*k["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in k else None
        res.append(dict(name=name, dram_read=rd, dram_write=wr,
                        time_ms=float(k["gpu__time_duration.sum"][0].replace(",", "")) *
                        (1e-3 if k["gpu__time_duration.sum"][1] == "us" else
                         1e-6 if k["gpu__time_duration.sum"][1] == "ns" else 1)))
        lines.append("")
    return lines, res


def summarise_launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), \
        hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    hack = {n: t for n, t in tot.items() if any(s in n for s in ("hack", "prefill", "decode", "ingest", "append",
                                                                     "quant", "homomm", "gather", "scatter"))}
    total = sum(hack.values())
    lines = ["| kernel (libhack) | launches | total ms | share of libhack time |", "|---|---|---|---|"]
    for n, t in sorted(hack.items(), key=lambda x: -x[1]):
        lines.append(f"| `{n[:90]}` | {cnt[n]} | {t:.3f} | {100 * t / total:.1f}% |")
    return lines


def main():
    tag = sys.argv[1]
    out = os.path.join(ROOT, "gpurun_out")
    md = [f"# ncu summary `{tag}`\n",
          "Captured with `scripts/ncu_profile.sh` under gpurun on one B200 (`--clock-control none`). "
          "Launch times are cold-cache and serialised: compare shares, not absolutes.\n"]
    lp = os.path.join(out, f"{tag}_launches.csv")
    if os.path.exists(lp):
        md += ["## Launch list (bench.py --steps 2 --warmup 3)\n"] + summarise_launches(lp) + [""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for part, key in (("prefill", "prefill_attention"), ("decode", "decode_attention")):
        rep = os.path.join(out, f"{tag}_{part}.ncu-rep")
        if not os.path.exists(rep):
            continue
        lines, res = summarise_rep(rep)
        md += [f"## `ncu --set full`: {part} attention kernel\n"] + lines
        if res and res[0]["dram_read"] is not None:
            r = res[0]
            traffic[key] = {"dram_bytes_per_launch": r["dram_read"] + r["dram_write"], "kernel": r["name"][:120],
                            "source": f"profiles/{tag}.md", "ncu_time_ms": r["time_ms"]}
    open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
