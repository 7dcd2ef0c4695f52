"""ctypes binding of librqmc_b200.so (C ABI declared in include/rqmc_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1408_5526_b200/csrc``).  There is no fallback: if the
library is missing or no CUDA device is present, every device entry point
raises.  Error codes map onto the reference's exception types
(harness.py:28-29 ConfigurationError/ValueError, harness.py:222-226
ArithmeticError).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
# RQMC_B200_LIB: alternative build of the same ABI (A/B kernel experiments)
LIB_PATH = Path(os.environ.get("RQMC_B200_LIB", HERE / "librqmc_b200.so"))

RQ_OK, RQ_ERR_VALUE, RQ_ERR_CUDA, RQ_ERR_RANGE, RQ_ERR_NONFINITE = 0, -1, -2, -3, -4

GEN_IDS = {
    "rasrap-recursive": 0,
    "rasrap-counter": 1,
    "philox": 2,
    "sobol-gray": 3,
    "sobol-counter": 4,
    "sfc64": 5,
    "twister": 6,
    "xorwow": 7,
    "kakutani": 8,
}
MODEL_IDS = {"libor": 0, "mbs": 1, "x1": 2, "const1": 3, "xhash": 5}

# kernels each ABI call launches when it succeeds are counted by the library
# itself (rq_estimate / rq_run_replications kernel_launches argument).


class RqModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_int32),
        ("delta", C.c_double),
        ("sigma", C.c_double),
        ("strike", C.c_double),
        ("front_factor", C.c_double),
        ("i0", C.c_double),
        ("k0", C.c_double),
        ("k1", C.c_double),
        ("k2", C.c_double),
        ("k3", C.c_double),
        ("k4", C.c_double),
        ("sigma_xi", C.c_double),
        ("payment", C.c_double),
        ("table", C.POINTER(C.c_double)),
    ]


class DeviceError(RuntimeError):
    """A CUDA / driver failure inside librqmc_b200."""


_lib = None


def _declare(L):
    P, vp = C.POINTER, C.c_void_p
    i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
    L.rq_last_error.restype = C.c_char_p
    L.rq_abi_version.restype = C.c_int
    L.rq_sampler_create.argtypes = [P(vp), C.c_int, C.c_int, u64, i64, i32, vp]
    L.rq_sampler_destroy.argtypes = [vp]
    L.rq_sampler_destroy.restype = None
    L.rq_sampler_points.argtypes = [vp, i32, i64, i64, vp, vp]
    L.rq_sampler_points_at.argtypes = [vp, i32, vp, i64, vp, vp]
    L.rq_index_limit.restype = i64
    L.rq_index_limit.argtypes = [C.c_int]
    L.rq_sampler_rasrap_tables.argtypes = [vp, i32, vp, vp, vp]
    L.rq_estimate.argtypes = [vp, P(RqModel), P(i64), i32, vp, P(i32), vp]
    L.rq_run_replications.argtypes = [C.c_int, P(RqModel), u64, i64, i64, P(i64), i32, P(dbl),
                                      P(i32)]
    L.rq_model_payoffs.argtypes = [P(RqModel), vp, i64, vp, vp]
    L.rq_inv_normal.argtypes = [vp, i64, vp, vp]
    L.rq_stream_normals.argtypes = [vp, i32, i64, vp, vp, vp]
    L.rq_pairwise_sum.argtypes = [vp, i64, vp, vp]
    L.rq_pairwise_sum_host.argtypes = [P(dbl), i64, P(dbl)]
    L.rq_stats_reset.argtypes = [C.c_int]
    L.rq_stats_reset.restype = None
    L.rq_stats_get.argtypes = [P(C.c_uint64), P(C.c_uint64), P(dbl), P(dbl), P(dbl), P(i64)]
    L.rq_stats_get.restype = None
    L.rq_fp64_peak.argtypes = [P(dbl), P(dbl)]
    L.rq_sobol_directions.argtypes = [C.c_int, P(C.c_uint32)]
    L.rq_halton_constants.argtypes = [C.c_int, P(C.c_int32), P(C.c_int32), P(dbl)]
    L.rq_halton_divide.argtypes = [C.c_int, u64, P(u64), P(C.c_uint32)]
    L.rq_kakutani_tables.argtypes = [C.c_int, P(dbl), P(dbl)]
    for name in ("rq_sampler_create", "rq_sampler_points", "rq_sampler_points_at",
                 "rq_sampler_rasrap_tables", "rq_estimate", "rq_run_replications",
                 "rq_model_payoffs", "rq_inv_normal", "rq_stream_normals", "rq_pairwise_sum",
                 "rq_pairwise_sum_host", "rq_fp64_peak",
                 "rq_sobol_directions", "rq_halton_constants", "rq_halton_divide",
                 "rq_kakutani_tables"):
        getattr(L, name).restype = C.c_int


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() or "
                "`make -C paper_1408_5526_b200/csrc` (there is no CPU fallback)"
            )
        L = C.CDLL(str(LIB_PATH))
        _declare(L)
        if L.rq_abi_version() != 1:
            raise ImportError("librqmc_b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == RQ_OK:
        return
    msg = (lib().rq_last_error() or b"").decode()
    if rc in (RQ_ERR_VALUE, RQ_ERR_RANGE):
        from .harness import ConfigurationError

        raise ConfigurationError(msg)
    if rc == RQ_ERR_NONFINITE:
        raise ArithmeticError(msg)
    raise DeviceError(msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("paper_1408_5526_b200 needs a CUDA device (no CPU fallback)")
    return torch


def stream_ptr():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def model_struct(model) -> tuple[RqModel, object]:
    """Pack a LiborModel / MbsModel / test model into the ABI struct.

    Returns (struct, keepalive) -- keepalive owns the host table memory.
    """
    import numpy as np

    m = RqModel()
    m.kind = MODEL_IDS[model.name]
    m.dim = int(model.dim)
    keep = None
    if model.name == "libor":
        c = model.config
        m.delta, m.sigma, m.strike = c.accrual, c.sigma, c.strike
        m.front_factor = 1.0 / (1.0 + c.accrual * model.front_rate)  # models.py:320
        keep = np.ascontiguousarray(model.initial_rates, dtype=np.float64)
    elif model.name == "mbs":
        c = model.config
        m.i0, m.k0, m.k1, m.k2, m.k3, m.k4 = c.initial_rate, c.k0, c.k1, c.k2, c.k3, c.k4
        m.sigma_xi, m.payment = c.sigma_xi, c.payment
        keep = np.ascontiguousarray(model.annuity, dtype=np.float64)
    if keep is not None:
        m.table = keep.ctypes.data_as(C.POINTER(C.c_double))
    return m, keep


def stats_reset(timing: bool = False) -> None:
    lib().rq_stats_reset(1 if timing else 0)


def stats_get() -> dict:
    h2d, d2h = C.c_uint64(), C.c_uint64()
    su, pa, re = C.c_double(), C.c_double(), C.c_double()
    n = C.c_int64()
    lib().rq_stats_get(C.byref(h2d), C.byref(d2h), C.byref(su), C.byref(pa), C.byref(re),
                       C.byref(n))
    return {"h2d": h2d.value, "d2h": d2h.value, "setup_ms": su.value, "paths_ms": pa.value,
            "reduce_ms": re.value, "paths_launches": n.value}


def fp64_peak() -> tuple[float, float]:
    """(DFMA slots/s over all SMs, best kernel ms) from the on-device probe."""
    r, ms = C.c_double(), C.c_double()
    check(lib().rq_fp64_peak(C.byref(r), C.byref(ms)))
    return r.value, ms.value
