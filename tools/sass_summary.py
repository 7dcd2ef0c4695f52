"""SASS instruction counts per kernel of librqmc_b200.so (cuobjdump -sass):
total, local-memory spill traffic (LDL/STL), DFMA/DMUL/DADD and MUFU.RCP64H.

    python tools/sass_summary.py [lib.so] > profiles/<round>_sass_summary.txt
"""
import re
import subprocess
import sys
from collections import Counter

so = sys.argv[1] if len(sys.argv) > 1 else "paper_1408_5526_b200/librqmc_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in txt.split("\n"):
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and cur:
        op = m.group(2)
        c = counts[cur]
        c["insts"] += 1
        base = op.split(".")[0]
        if base in ("LDL", "STL"):
            c["LDL/STL"] += 1
        if base in ("DFMA", "DMUL", "DADD"):
            c[base] += 1
        if op.startswith("MUFU.RCP64H"):
            c["MUFU.RCP64H"] += 1
print(f"SASS instruction counts per kernel ({so}, sm_100a; cuobjdump -sass)")
print(f"{'insts':>7s} {'LDL/STL':>7s} {'DFMA':>5s} {'DMUL':>5s} {'DADD':>5s} {'RCP64H':>6s}  function")
tot_spill = 0
for f, c in counts.items():
    if not c["insts"]:
        continue
    tot_spill += c["LDL/STL"]
    print(f"{c['insts']:7d} {c['LDL/STL']:7d} {c['DFMA']:5d} {c['DMUL']:5d} {c['DADD']:5d} "
          f"{c['MUFU.RCP64H']:6d}  {f}")
print(f"# {len([c for c in counts.values() if c['insts']])} kernels, {tot_spill} LDL/STL in total")
