"""Small calls through every device entry point (run under compute-sanitizer)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_5526_b200 import models as M  # noqa: E402
from paper_1408_5526_b200.harness import estimate_replications  # noqa: E402
from paper_1408_5526_b200.samplers import DeviceSampler  # noqa: E402

for gen in ("rasrap-recursive", "rasrap-counter", "philox", "sobol-gray", "sobol-counter", "sfc64"):
    for dim in (2, 20, 80, 360):
        s = DeviceSampler(gen, dim, 20120224, 3)
        a = s.points(0, 300)
        b = s.points(1000, 257)
        c = s.points_at(np.array([0, 5, 2**20 + 3, 2**32 - 1]))
        torch.cuda.synchronize()
    for model in (M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)),
                  M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25)), M.MbsModel(),
                  M.FirstCoordinateModel()):
        th = estimate_replications(gen, model, 20120224, 1, 2, (100, 1000))
        assert np.all(np.isfinite(th)), (gen, model.name)
print("sanitize smoke ok")
