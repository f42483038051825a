#!/usr/bin/env python3
"""Summarise ncu output for profiles/ (committed evidence).

    python tools/ncu_summary.py full  <report.ncu-rep> <kernel-key> [--out profiles/ncu_summary.json]
    python tools/ncu_summary.py launches <launches.csv> [--out profiles/...json]

`full` extracts, per profiled launch, duration, DRAM bytes (read + write),
L2 hit rate, achieved occupancy, issue activity, fp64 pipe use and the top
stall reasons, and merges them into the JSON under <kernel-key> (bench.py
reads "dram_bytes_per_launch" from there for roofline.traffic). `launches`
turns the gpu__time_duration launch list into per-kernel shares.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
    "instructions": ("smsp__inst_executed.sum", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
              "ns": 1, "us": 1e3, "ms": 1e6}


def fnum(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def full(report: str, key: str, out: Path) -> None:
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:160]}
        for name, (metric, _) in KEYS.items():
            if metric not in d:
                continue
            v = fnum(d[metric])
            unit = u.get(metric, "")
            if name.startswith("dram_") and name.endswith("bytes"):
                v *= UNIT_SCALE.get(unit, 1)
            if name == "duration_us":
                v = v * UNIT_SCALE.get(unit, 1) / 1e3
            rec[name] = v
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): fnum(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        launches.append(rec)
    summary = json.loads(out.read_text()) if out.exists() else {}
    dram = [l["dram_read_bytes"] + l["dram_write_bytes"] for l in launches if "dram_read_bytes" in l]
    summary[key] = {"report": Path(report).name, "launches": launches,
                    "dram_bytes_per_launch": sum(dram) / len(dram) if dram else None}
    out.write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary[key], indent=1))


def launch_list(path: str, out: Path) -> None:
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        per[r[ik].split("(")[0][:100]].append(fnum(r[iv]) * UNIT_SCALE.get(r[iu], 1) / 1e3)
    total = sum(sum(v) for v in per.values())
    res = {k: {"launches": len(v), "total_us": round(sum(v), 2), "mean_us": round(sum(v) / len(v), 2),
               "share_pct": round(100 * sum(v) / total, 1)} for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}
    out.write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["full", "launches"])
    ap.add_argument("path")
    ap.add_argument("key", nargs="?", default="")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    a = ap.parse_args()
    out = Path(a.out)
    out.parent.mkdir(exist_ok=True)
    if a.mode == "full":
        full(a.path, a.key, out)
    else:
        launch_list(a.path, out)


if __name__ == "__main__":
    main()
