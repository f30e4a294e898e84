"""Summarise ncu output into profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <prof.ncu-rep> <out.md> [--traffic-key KEY]

`launches`: per-kernel share of the device time from a
`ncu --metrics gpu__time_duration.sum --clock-control none` launch list.
`full`: key metrics of a `ncu --set full` capture; with --traffic-key also
records dram read+write bytes per launch into profiles/traffic.json (the
`roofline.traffic` field bench.py reports).
"""

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(src, out, split=None):
    """split = (substring, threshold_us, label): launches of a kernel whose name
    contains `substring` and that run longer than the threshold are listed
    separately (bench.py's zero-copy e2e sync launches read host memory over
    PCIe and take milliseconds; the device-resident ones ~100 us)."""
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1)
            key = r[ki]
            if split and split[0] in key and v > split[1]:
                key = f"{key} [{split[2]}]"
            agg[key].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# launch list: {Path(src).name}", "",
             "| launches | total us | share | avg us | kernel |", "|---:|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        name = k if len(k) <= 110 else (k[:110] + (k[k.rindex(" ["):] if k.endswith("]") else ""))
        lines.append(f"| {len(v)} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% | {sum(v) / len(v):.2f} | `{name}` |")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(src, out, traffic_key=None):
    txt = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full: {Path(src).name}", ""]
    per_launch = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines.append(f"## launch {r[h.index('ID')]}: `{name[:120]}`")
        lines.append("| metric | unit | value |")
        lines.append("|---|---|---:|")
        for k in KEYS:
            if k in h:
                lines.append(f"| {k} | {units[h.index(k)]} | {r[h.index(k)]} |")
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * SCALE.get(units[h.index("dram__bytes_read.sum")], 1)
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * SCALE.get(units[h.index("dram__bytes_write.sum")], 1)
        per_launch.append(rd + wr)
        lines.append(f"| dram read+write | byte | {rd + wr:.0f} |")
        lines.append("")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_key and per_launch:
        tp = ROOT / "profiles" / "traffic.json"
        d = json.loads(tp.read_text()) if tp.exists() else {}
        d[traffic_key] = sum(per_launch) / len(per_launch)
        tp.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    mode, src, out = sys.argv[1:4]
    if mode == "launches":
        sp = None
        if "--split" in sys.argv:  # --split SUBSTRING THRESHOLD_US LABEL
            i = sys.argv.index("--split")
            sp = (sys.argv[i + 1], float(sys.argv[i + 2]), sys.argv[i + 3])
        launches(src, out, sp)
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(src, out, key)
