"""One small fused-path estimate for ncu (warm-up call + profiled call).

    ncu --set full -k regex:k_paths -s 1 -c 1 -o gpurun_out/prof \
        python tools/profile_step.py --workload c2 --reps 8
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--generator", default="rasrap-recursive")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_1408_5526_b200.harness import estimate_replications

    kind, mat, acc, M, N, _ = bench.WORKLOADS[a.workload]
    model = bench.build_model(kind, mat, acc)
    n = a.n or N
    for _ in range(2):
        th = estimate_replications(a.generator, model, bench.SEED, 1, a.reps, (n,))
    torch.cuda.synchronize()
    print("theta[0] =", th[0, 0])


if __name__ == "__main__":
    main()
