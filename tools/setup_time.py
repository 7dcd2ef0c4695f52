"""Time rq_sampler_create (device randomisation setup) for Rasrap samplers."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1408_5526_b200 import _lib  # noqa: E402

lib = _lib.lib()
torch.cuda.init()
st = _lib.stream_ptr()
for dim, reps in ((20, 1), (360, 1), (360, 256), (1000, 1), (6542, 1)):
    for gen in ("rasrap-recursive", "sobol-gray", "philox"):
        if gen == "sobol-gray" and dim > 421:
            continue
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = C.c_void_p()
            _lib.check(lib.rq_sampler_create(C.byref(h), _lib.GEN_IDS[gen], dim, 20120224, 1, reps,
                                             st))
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            lib.rq_sampler_destroy(h)
        print(f"{gen:18s} dim {dim:5d} reps {reps:4d}: create+setup {min(ts[1:]):8.3f} ms")
