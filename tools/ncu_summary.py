"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch CSVs) into profiles/.

    python tools/ncu_summary.py r1     # -> profiles/r1_ncu_summary.md + .json
"""

from __future__ import annotations

import csv
import glob
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "inst",
}
SASS_EVIDENCE = ("UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "HMMA", "FFMA2",
                 "FADD2", "FMNMX3", "MUFU.EX2")


def raw_metrics(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    hdr, unit, val = rows[0], rows[1], rows[2]
    out = {"kernel": val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for h, u, v in zip(hdr, unit, val):
        if h in METRICS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if u == "Gbyte":
                x *= 1e9
            elif u == "Mbyte":
                x *= 1e6
            elif u == "Kbyte":
                x *= 1e3
            elif u == "us":
                x *= 1e3
            elif u == "ms":
                x *= 1e6
            out[METRICS[h]] = x  # bytes, ns
    return out


def sass_counts(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    import re

    counts = defaultdict(int)
    for line in txt.splitlines():
        for tok in re.findall(r"\b[A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*", line):
            base = tok.split(".")[0]
            for m in SASS_EVIDENCE:
                if tok == m or base == m or (m.startswith(base) and tok.startswith(m)):
                    counts[m] += 1
    return dict(counts)


def launch_shares(path: str) -> list:
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
            name = name.split("(")[0].split("<")[0].strip()
            v = float(d["Metric Value"].replace(",", ""))
            if d["Metric Unit"] == "us":
                v *= 1e3
            elif d["Metric Unit"] == "ms":
                v *= 1e6
            tot[name] += v
            cnt[name] += 1
    grand = sum(tot.values()) or 1.0
    return sorted(({"kernel": k, "launches": cnt[k], "total_ms": tot[k] / 1e6,
                    "share": tot[k] / grand} for k in tot), key=lambda x: -x["total_ms"])


def main(tag: str) -> None:
    res = {"kernels": {}, "launches": None}
    for rep in sorted(glob.glob(os.path.join(OUT, f"{tag}_*.ncu-rep"))):
        name = os.path.basename(rep)[len(tag) + 1:-len(".ncu-rep")]
        m = raw_metrics(rep)
        m["sass"] = sass_counts(rep)
        if "dram_read" in m:
            m["dram_traffic_bytes"] = m["dram_read"] + m.get("dram_write", 0.0)
        res["kernels"][name] = m
    lpath = os.path.join(OUT, f"{tag}_bench_launches.csv")
    if os.path.exists(lpath):
        res["launches"] = launch_shares(lpath)
    prof = os.environ.get("PROFILES_DIR", os.path.join(ROOT, "profiles"))  # gpurun: gpurun_out
    os.makedirs(prof, exist_ok=True)
    json.dump(res, open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w"), indent=1)
    lines = [f"# ncu summary ({tag})", "",
             "Captures: `ncu --set full --clock-control none --import-source on` (one launch each, "
             "tools/ncu_capture.sh); numbers taken under ncu are profiles, not bench values.", "",
             "| capture | kernel | duration us | DRAM read MB | DRAM write MB | DRAM % | tensor % "
             "| SM % | regs | SASS evidence |", "|---|---|---|---|---|---|---|---|---|---|"]
    for name, m in res["kernels"].items():
        ev = ", ".join(f"{k}x{v}" for k, v in sorted(m.get("sass", {}).items()))
        lines.append(
            f"| {name} | `{m.get('kernel', '?')[:60]}` | {m.get('duration', 0) / 1e3:.1f} | "
            f"{m.get('dram_read', 0) / 1e6:.1f} | {m.get('dram_write', 0) / 1e6:.1f} | "
            f"{m.get('dram_pct', 0):.1f} | {m.get('tensor_pct', 0):.1f} | {m.get('sm_pct', 0):.1f} | "
            f"{int(m.get('regs', 0))} | {ev} |")
    if res["launches"]:
        lines += ["", "## Launch list of `bench.py --steps 2 --warmup 1` under ncu "
                  "(cold-cache, serialised: compare shares)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for r in res["launches"][:12]:
            lines.append(f"| `{r['kernel'][:70]}` | {r['launches']} | {r['total_ms']:.2f} | "
                         f"{100 * r['share']:.1f}% |")
    open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
