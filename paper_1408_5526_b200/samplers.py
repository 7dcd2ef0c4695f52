"""Device-backed samplers: one replication's randomised point stream.

Same protocol as the reference samplers (``dim``, ``counter_based``,
``fill(out)``, ``at(indices)``; halton.py:451-518, sobol.py:330-372,
harness.py:37-72).  The randomisation (Rasrap random starts and digit
permutations, Sobol' scrambles, Philox / SFC64 keys) is derived from
``(seed, family, replication)`` ON THE DEVICE by librqmc_b200.so, bit-identical
to the reference's numpy SeedSequence/PCG64 draws, and every point is
evaluated by a sm_100a kernel.  Points are bit-exact with the reference's
``fill`` / ``at`` for the same seed and replication.

``fill``/``at`` accept numpy arrays (host, copied back) or CUDA tensors
(written in place on the device).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

# generators whose points are pure functions of the index (harness.py:96);
# on the device every generator is evaluated per index, but the reference's
# attribute is kept so stride-parallel validation behaves the same.
COUNTER_BASED = frozenset({"philox", "rasrap-counter", "sobol-counter", "sfc64"})


class DeviceSampler:
    """Replication ``replication`` of generator ``name`` in ``dim`` dimensions."""

    def __init__(self, name: str, dim: int, seed: int, replication: int):
        torch = _lib.require_cuda()
        if name not in _lib.GEN_IDS:
            raise ValueError(f"generator {name!r} has no device implementation")
        self.name = name
        self.dim = int(dim)
        self.seed = int(seed)
        self.replication = int(replication)
        self.counter_based = name in COUNTER_BASED
        self._next = 0
        h = C.c_void_p()
        _lib.check(_lib.lib().rq_sampler_create(
            C.byref(h), _lib.GEN_IDS[name], self.dim, self.seed & 0xFFFFFFFFFFFFFFFF,
            self.replication, 1, _lib.stream_ptr()))
        self._h = h
        self._torch = torch

    def close(self) -> None:
        """Release the device tables now (also done when the object dies)."""
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._torch.cuda.current_stream().synchronize()
            _lib.lib().rq_sampler_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    # -- device-level API -------------------------------------------------
    def points(self, first: int, count: int):
        """CUDA tensor [count, dim] of points first..first+count-1."""
        torch = self._torch
        out = torch.empty((count, self.dim), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().rq_sampler_points(self._h, 0, int(first), int(count),
                                                 out.data_ptr(), _lib.stream_ptr()))
        return out

    def points_at(self, indices):
        torch = self._torch
        idx = torch.as_tensor(np.asarray(indices, dtype=np.int64) if not isinstance(
            indices, torch.Tensor) else indices, dtype=torch.int64).to("cuda").contiguous()
        if idx.numel() and int(idx.min()) < 0:
            raise ValueError("index must be non-negative")
        lim = int(_lib.lib().rq_index_limit(_lib.GEN_IDS[self.name]))
        if idx.numel() and int(idx.max()) >= lim:
            from .harness import ConfigurationError

            raise ConfigurationError(f"point index exceeds the device index range of "
                                     f"{self.name} ({lim})")
        out = torch.empty((idx.numel(), self.dim), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().rq_sampler_points_at(self._h, 0, idx.data_ptr(), idx.numel(),
                                                    out.data_ptr(), _lib.stream_ptr()))
        return out

    # -- reference protocol ---------------------------------------------
    # Sequential streams (MT19937, XORWOW, Kakutani) are positioned by
    # walking them from their start, so a call at point `first` costs
    # O(first); fill() reads ahead a block of up to READAHEAD_BYTES of points
    # and serves consecutive fills from it (repeated small fills, e.g. the
    # CLI's 8192-row blocks, are O(n) overall instead of O(n^2)).
    READAHEAD_BYTES = 256 << 20
    SEQUENTIAL = frozenset({"twister", "xorwow", "kakutani"})

    def fill(self, out) -> None:
        """Write the next ``len(out)`` points of the stream into ``out``."""
        n = int(out.shape[0])
        if self.name in self.SEQUENTIAL:
            pts = self._readahead(self._next, n)
        else:
            pts = self.points(self._next, n)
        self._next += n
        _store(out, pts)

    def _readahead(self, first: int, n: int):
        buf, b0 = getattr(self, "_ra", None), getattr(self, "_ra_first", 0)
        if buf is None or first < b0 or first + n > b0 + buf.shape[0]:
            rows = max(n, self.READAHEAD_BYTES // (8 * self.dim))
            lim = int(_lib.lib().rq_index_limit(_lib.GEN_IDS[self.name]))
            rows = max(n, min(rows, lim - first))
            self._ra, self._ra_first = self.points(first, rows), first
            buf, b0 = self._ra, first
        return buf[first - b0:first - b0 + n]

    def at(self, indices):
        if not self.counter_based:
            raise TypeError(f"{self.name} is not counter-based (use fill)")
        pts = self.points_at(indices)
        return pts if isinstance(indices, self._torch.Tensor) else pts.cpu().numpy()

    def rasrap_tables(self):
        """(start digits, sigma values, init partial sums) of this replication."""
        from .tables import halton_layout

        lay = halton_layout(self.dim)
        dig = np.empty(((lay["caps"] + 3) & ~3), dtype=np.uint16)
        sig = np.empty(((lay["bases"] + 3) & ~3), dtype=np.uint16)
        sums = np.empty(lay["sums"], dtype=np.float64)
        _lib.check(_lib.lib().rq_sampler_rasrap_tables(
            self._h, 0, dig.ctypes.data, sig.ctypes.data, sums.ctypes.data))
        return dig, sig, sums


def _store(out, pts) -> None:
    torch = pts.__class__.__module__.startswith("torch") and __import__("torch")
    if torch is not None and isinstance(out, torch.Tensor):
        out.copy_(pts)
    else:
        out[...] = pts.cpu().numpy()
