"""Registers / spills / smem per kernel from the ptxas -v log of the csrc build.

    python tools/ptxas_regs.py [paper_1408_5526_b200/csrc/ptxas.log] [filter]
"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] else "paper_1408_5526_b200/csrc/ptxas.log"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = []
for ln in open(log):
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = {"name": m.group(1)}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        cur["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers.*?(?:(\d+) bytes smem)?$", ln.strip())
    if m:
        cur["regs"] = int(m.group(1))
        cur["smem"] = int(m.group(2) or 0)
        rows.append(cur)
        cur = None
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.split("\n")
for r, n in zip(rows, names):
    if flt in n:
        print(f"{r['regs']:4d} regs {r.get('spill', 0):4d} spill {r['smem']:6d} smem  {n[:110]}")
