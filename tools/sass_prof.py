"""Join an ncu per-SASS-instruction CSV (--page source --print-source=sass)
with `nvdisasm -g` line info of the same kernel, and print instruction and
stall totals per source line and per named region.

    python tools/sass_prof.py sass.csv.gz librqmc_b200.so KERNEL_MANGLED [--lines 40]
"""
import csv
import gzip
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

# (file, first line, last line, region) -- rq_kernels.cu / rq_device.cuh
REGIONS = []


def load_regions(src: Path):
    """Region = the enclosing struct/function of each line (brace-level scan)."""
    regs = []
    for f in ("rq_kernels.cu", "rq_device.cuh"):
        lines = (src / f).read_text().split("\n")
        cur = None
        for i, l in enumerate(lines, 1):
            m = re.match(r"^(?:template <[^>]*>\s*)?(?:struct|__global__|__device__|static|__host__)\s.*?([A-Za-z_][A-Za-z0-9_]*)\s*[({]", l)
            if m and not l.startswith(" "):
                cur = m.group(1)
            m2 = re.match(r"^  (?:__device__|static __device__|__host__ __device__)[^;]*?([A-Za-z_][A-Za-z0-9_]*)\(", l)
            name = cur
            if m2:
                name = f"{cur}::{m2.group(1)}"
                regs.append((f, i, m2.group(1)))
            elif m:
                regs.append((f, i, cur))
        # keep
    out = defaultdict(list)
    for f, i, n in regs:
        out[f].append((i, n))
    return out


def region_of(regs, f, ln):
    best = "?"
    for i, n in regs.get(f, []):
        if i <= ln:
            best = n
        else:
            break
    return best


def sass_lines(so: str, kernel: str):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(so).resolve())], cwd=d, capture_output=True)
        cub = [p for p in Path(d).glob("*.cubin") if "capi" not in p.name][0]
        txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout
    lines = txt.split("\n")
    i = lines.index(f".text.{kernel}:")
    out, cur = [], ("?", 0)
    for l in lines[i + 1:]:
        if l.startswith("//----"):
            break
        if "//## File" in l:
            cur = (l.split('"')[1].split("/")[-1], int(l.split("line")[1].split(",")[0]))
            continue
        if "/*" in l and ";" in l:
            out.append((cur, l.split("*/", 1)[1].strip()))
    return out


def main():
    csvp, so, kernel = sys.argv[1:4]
    nl = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 40
    raw = gzip.open(csvp, "rt").read() if csvp.endswith(".gz") else open(csvp).read()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    sl = sass_lines(so, kernel)
    if len(sl) != len(data):
        print(f"warning: {len(sl)} disassembled vs {len(data)} profiled instructions")
    regs = load_regions(Path(__file__).resolve().parents[1] / "paper_1408_5526_b200" / "csrc")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_line = defaultdict(lambda: defaultdict(float))
    by_reg = defaultdict(lambda: defaultdict(float))
    tot = defaultdict(float)
    for (loc, ins), d in zip(sl, data):
        ie = float(d["Instructions Executed"] or 0)
        op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
        fp64 = op.startswith(("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
        reg = region_of(regs, *loc)
        for tgt in (by_line[loc], by_reg[reg], tot):
            tgt["inst"] += ie
            tgt["fp64"] += ie if fp64 else 0
            tgt["samples"] += float(d["Warp Stall Sampling (All Samples)"] or 0)
            for s in stalls:
                tgt[s] += float(d[s] or 0)
    T, S = tot["inst"], tot["samples"]
    top = sorted(stalls, key=lambda s: -tot[s])[:6]
    print(f"total warp instructions {T:.4g}, fp64 share {tot['fp64'] / T:.3f}, samples {S:.0f}")
    print("stall mix:", ", ".join(f"{s[6:]} {tot[s] / S:.2f}" for s in top))
    hdrl = f"{'region':40s} {'inst%':>6s} {'fp64%':>6s} {'samp%':>6s} " + " ".join(f"{s[6:12]:>7s}" for s in top)
    print("\n" + hdrl)
    for r, v in sorted(by_reg.items(), key=lambda kv: -kv[1]["inst"]):
        if v["inst"] / T < 0.002:
            continue
        print(f"{r[:40]:40s} {v['inst'] / T * 100:6.1f} {v['fp64'] / max(v['inst'], 1) * 100:6.1f} "
              f"{v['samples'] / S * 100:6.1f} " + " ".join(f"{v[s] / S * 100:7.2f}" for s in top))
    print("\n" + f"{'line':28s} {'inst%':>6s} {'samp%':>6s} " + " ".join(f"{s[6:12]:>7s}" for s in top))
    for loc, v in sorted(by_line.items(), key=lambda kv: -kv[1]["samples"])[:nl]:
        print(f"{loc[0][:18]:18s}:{loc[1]:<9d} {v['inst'] / T * 100:6.2f} {v['samples'] / S * 100:6.2f} "
              + " ".join(f"{v[s] / S * 100:7.2f}" for s in top))


if __name__ == "__main__":
    main()
