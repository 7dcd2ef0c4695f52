"""Helper for test_host.py: run under torchrun (gloo, CPU) -- the sharded
replication path with the oracle standing in for the device estimator."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1408_5526_b200 import distributed as D  # noqa: E402
from paper_1408_5526_b200 import models as M  # noqa: E402


def est(gen, model, seed, first, count, grid):
    return O.run_replications(gen, model, seed, first, count, grid, threads=2)


dist.init_process_group("gloo")
model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
theta = D.estimate_sharded("philox", model, 20120224, 7, (1000, 4096), estimator=est)
world = dist.get_world_size()
if dist.get_rank() == 0:
    print(json.dumps({"world": world, "counts": [D.shard(7, world, r)[1] for r in range(world)],
                      "theta": theta.tolist()}))
dist.destroy_process_group()
