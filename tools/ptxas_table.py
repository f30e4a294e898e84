"""Per-kernel registers / spills from paper_2507_09029_b200/_lib/ptxas.log.

    python tools/ptxas_table.py [substring]
"""
import re
import subprocess
import sys
from pathlib import Path

log = (Path(__file__).resolve().parent.parent / "paper_2507_09029_b200" / "_lib" / "ptxas.log").read_text()
pat = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for ln in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", ln)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        rows.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        rows.setdefault(cur, {})["regs"] = m.group(1)
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    if pat in d:
        r = rows[n]
        print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', '?'):>9}  {d[:100]}")
