"""Small calls through every device entry point (run under compute-sanitizer).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_smoke.py [quick]

Covers every generator (the sequential MT19937 / XORWOW / Kakutani streams
included), the points / at / estimate / stream (store and store-less) / payoff
/ inverse-normal entry points, the warp-specialised path kernel (Rasrap +
LIBOR S=20), multi-batch estimates (RQ_BATCH_PATHS forces several payoff
batches so the reduction's last-block ticket folding runs per batch) and the
multi-chunk Rasrap stream (per-chunk atomic run counters).  Sizes are tiny:
the sanitizers slow kernels down by 10-100x.
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("RQ_BATCH_PATHS", "2048")  # several payoff batches per estimate

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_5526_b200 import _lib  # noqa: E402
from paper_1408_5526_b200 import models as M  # noqa: E402
from paper_1408_5526_b200.harness import estimate_replications  # noqa: E402
from paper_1408_5526_b200.samplers import DeviceSampler  # noqa: E402

QUICK = len(sys.argv) > 1 and sys.argv[1] == "quick"
SEED = 20120224
COUNTER = ("rasrap-recursive", "rasrap-counter", "philox", "sobol-gray", "sobol-counter", "sfc64")
SEQ = ("twister", "xorwow", "kakutani")
dims = (2, 20, 360) if QUICK else (2, 20, 80, 360)

for gen in COUNTER + SEQ:
    for dim in dims:
        s = DeviceSampler(gen, dim, SEED, 3)
        s.points(0, 300)
        s.points(1000, 257)
        if gen in COUNTER:
            s.points_at(np.array([0, 5, 2**20 + 3, 2**32 - 1]))
        torch.cuda.synchronize()
        s.close()
    models = [M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)), M.MbsModel(),
              M.CoordinateHashModel(20)]
    if not QUICK:
        models += [M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25)),
                   M.FirstCoordinateModel()]
    for model in models:
        th = estimate_replications(gen, model, SEED, 1, 3, (100, 1000, 4100))
        assert np.all(np.isfinite(th)), (gen, model.name)

# config-4 stream: store and store-less, ragged point counts, multi-chunk Rasrap
out = torch.empty(1, dtype=torch.float64, device="cuda")
for gen in COUNTER:
    for dim, npts in ((360, 700), (7, 999)):
        s = DeviceSampler(gen, dim, SEED, 0)
        store = torch.empty((npts, dim), dtype=torch.float64, device="cuda")
        for dst in (store, None):
            _lib.check(_lib.lib().rq_stream_normals(s._h, 0, npts, out.data_ptr(),
                                                     dst.data_ptr() if dst is not None else None,
                                                     _lib.stream_ptr()))
        torch.cuda.synchronize()
        s.close()

# dims past the constant bank (global HaltonDim / Kakutani state) and LIBOR
# past the shared-memory model (per-CTA rate state in global memory)
for gen in ("rasrap-recursive", "rasrap-counter", "kakutani"):
    s = DeviceSampler(gen, 600, SEED, 1)
    s.points(0, 130)
    torch.cuda.synchronize()
    s.close()
big = M.LiborModel(M.LiborConfig(maturity=25.0, accrual=0.125))
for gen in ("rasrap-recursive", "philox", "xorwow"):
    th = estimate_replications(gen, big, SEED, 1, 2, (300,))
    assert np.all(np.isfinite(th)), gen
big.payoffs(np.random.default_rng(2).random((300, big.dim)))

# model payoffs and the scalar inverse normal from caller uniforms
u = np.random.default_rng(1).random((257, 20))
M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)).payoffs(u)
M.MbsModel(M.MbsConfig(months=20)).payoffs(u)
M.inv_normal(u.ravel())
torch.cuda.synchronize()
# torch's own blocks go back before the leak check (the library frees its
# allocations on every path; what remains would be torch's pinned staging)
del out, store
torch.cuda.synchronize()
torch.cuda.empty_cache()
print("sanitize smoke ok")
