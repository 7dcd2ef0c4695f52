"""Helper for test_gpu_benchsize.py: run under torchrun (gloo, ranks sharing
the visible GPU(s)) -- the sharded replication path with the DEVICE
estimator (distributed.estimate_sharded binds LOCAL_RANK mod #GPUs)."""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1408_5526_b200 import distributed as D  # noqa: E402
from paper_1408_5526_b200 import models as M  # noqa: E402

dist.init_process_group("gloo")
model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
theta = D.estimate_sharded("rasrap-recursive", model, 20120224, 37, (1000, 2**17))
if dist.get_rank() == 0:
    h = hashlib.sha256(np.ascontiguousarray(theta).tobytes()).hexdigest()
    print(json.dumps({"world": dist.get_world_size(), "sha": h, "theta": theta.tolist()}))
dist.destroy_process_group()
