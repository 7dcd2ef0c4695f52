"""Markdown table of a bench sweep (gpurun_out/sweep.json) for BASELINE.md §5."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
print("| Config | Generator | B200 value | frac (conv.) | e2e | CPU baseline (cores) | clock MHz |")
print("|---|---|---|---|---|---|---|")
for d in rows:
    c = d.get("config", {})
    r = d.get("roofline", {})
    e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    impl = d.get("impl", "ours")
    wl = c.get("workload", "")[:60]
    if impl == "reference":
        wl = "reference arm: " + wl
    val = f"{d['value']:.3e} {d['unit']}"
    fr = f"{r['frac']:.3f}" if r.get("frac") is not None else "—"
    e2 = f"{e['value']:.3e}" if e.get("value") and impl != "reference" else "—"
    cpu = f"{cb['value']:.3e} ({cb.get('cores')})" if cb else "—"
    clk = (d.get("clocks") or {}).get("sm_mhz")
    print(f"| {wl} | {c.get('generator', '')} | {val} | {fr} | {e2} | {cpu} | {clk} |")
