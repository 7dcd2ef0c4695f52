"""One line per bench.py JSON record: workload, generator, value, frac, kernel ms."""
import json
import sys

for ln in open(sys.argv[1]):
    ln = ln.strip()
    if not ln.startswith("{"):
        continue
    d = json.loads(ln)
    r = d.get("roofline", {})
    c = d.get("config", {})
    print(f"{c.get('workload', '')[:40]:40s} {c.get('generator', ''):17s} {d['value']:.4e} {d['unit']:10s}"
          f" frac {r.get('frac', 0):.3f} ms/step {d['ms_per_step']:.2f} clk {d.get('clocks', {}).get('sm_mhz')}")
