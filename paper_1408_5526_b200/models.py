"""Pricing models with device payoffs: LIBOR caplet and MBS.

Mirrors the reference's ``rqmcbench.models`` interface
(/root/reference/pkg/src/rqmcbench/models.py): ``LiborConfig``,
``LiborModel`` (``.dim``, ``.payoffs(u)``, ``.black_price()``),
``MbsConfig``, ``MbsModel``, ``ConstantModel``, ``FirstCoordinateModel``,
``inv_normal``, the yield-curve setup and the Black formula.

Model SETUP (spline yields, bonds, initial forwards, annuity ratios) is a
few dozen host scalars computed exactly as the reference does; the per-path
work (``payoffs`` and the fused engine in ``harness.run_experiment``) runs
in the sm_100a kernels of librqmc_b200.so.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.interpolate import CubicSpline

from . import _lib

# 2012-02-24 U.S. Treasury par curve (paper Table 3; reference
# data/treasury_2012-02-24.csv): tenor in years, yield in percent.
TREASURY_2012_02_24 = (
    (1.0 / 12.0, 0.08), (0.25, 0.10), (0.5, 0.14), (1.0, 0.18), (2.0, 0.31), (3.0, 0.43),
    (5.0, 0.89), (7.0, 1.41), (10.0, 1.98), (20.0, 2.75), (30.0, 3.10),
)


# ---------------------------------------------------------------- device helpers
def _as_device(u, dtype=None):
    """(tensor on cuda, was_host) for a numpy array or torch tensor."""
    torch = _lib.require_cuda()
    if isinstance(u, torch.Tensor):
        t = u.to(device="cuda", dtype=torch.float64).contiguous()
        return t, False
    arr = np.ascontiguousarray(u, dtype=np.float64)
    return torch.from_numpy(arr).to("cuda"), True


def inv_normal(u):
    """Standard normal quantile of the reference (models.py:73-82) on the GPU.

    Same two-branch rational approximation and 2**-53 clamp; evaluated with
    FMA Horner and a Newton reciprocal instead of the reference's two-rounding
    Horner and IEEE division, so results agree with the reference to within
    2e-13 * max(1, |x|) (the tested bar, tests/test_gpu_parity.py INVN_TOL);
    typically a few ulp.
    Accepts scalars, numpy arrays (returned as numpy) or CUDA tensors.
    """
    torch = _lib.require_cuda()
    scalar = np.ndim(u) == 0 and not isinstance(u, torch.Tensor)
    t, host = _as_device(np.atleast_1d(u) if scalar else u)
    out = torch.empty_like(t)
    _lib.check(_lib.lib().rq_inv_normal(t.data_ptr(), t.numel(), out.data_ptr(),
                                         _lib.stream_ptr()))
    if scalar:
        return float(out.cpu()[0])
    return out.cpu().numpy() if host else out


def norm_cdf(x: float) -> float:
    """Standard normal CDF via erfc (models.py:85-87)."""
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


# ---------------------------------------------------------------- yield curve
@dataclass(frozen=True)
class YieldCurve:
    """Treasury-style par yields: tenors in years, rates in percent (models.py:95-112)."""

    tenors: np.ndarray
    rates: np.ndarray
    _spline: CubicSpline = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        t = np.asarray(self.tenors, dtype=np.float64)
        r = np.asarray(self.rates, dtype=np.float64)
        if t.size != r.size or t.size < 2:
            raise ValueError("need matching tenor/rate arrays of length >= 2")
        if t[0] <= 0 or np.any(np.diff(t) <= 0):
            raise ValueError("tenors must be positive and strictly increasing")
        object.__setattr__(self, "tenors", t)
        object.__setattr__(self, "rates", r)
        object.__setattr__(self, "_spline", CubicSpline(t, r, bc_type="natural"))


def load_yield_curve(path) -> YieldCurve:
    """Read a ``tenor_years,rate_percent`` CSV (models.py:115-125)."""
    import csv

    tenors, rates = [], []
    with open(path, newline="") as f:
        reader = csv.DictReader(f)
        if reader.fieldnames != ["tenor_years", "rate_percent"]:
            raise ValueError(f"{path}: expected header tenor_years,rate_percent")
        for row in reader:
            tenors.append(float(row["tenor_years"]))
            rates.append(float(row["rate_percent"]))
    return YieldCurve(np.array(tenors), np.array(rates))


def default_curve() -> YieldCurve:
    t, r = zip(*TREASURY_2012_02_24)
    return YieldCurve(np.array(t), np.array(r))


def spline_rate(curve: YieldCurve, t: float) -> float:
    """Natural-cubic-spline yield (percent) at t, no extrapolation (models.py:136-142)."""
    if not curve.tenors[0] <= t <= curve.tenors[-1]:
        raise ValueError(f"t={t} outside curve range [{curve.tenors[0]}, {curve.tenors[-1]}]")
    return float(curve._spline(t))


def bond_prices(curve: YieldCurve, accrual: float, horizon: float) -> np.ndarray:
    """B(0, n*accrual) = exp(-y/100 * T), n = 1..horizon/accrual (models.py:145-156)."""
    count = round(horizon / accrual)
    if abs(count * accrual - horizon) > 1e-9:
        raise ValueError("horizon must be an integer number of accrual periods")
    times = accrual * np.arange(1, count + 1)
    ys = np.array([spline_rate(curve, t) for t in times]) / 100.0
    return np.exp(-ys * times)


def init_libor(bonds: np.ndarray, accrual: float) -> np.ndarray:
    """L_n(0) = (B_n - B_{n+1}) / (accrual B_{n+1}) (models.py:159-164)."""
    b = np.asarray(bonds, dtype=np.float64)
    if np.any(b <= 0):
        raise ValueError("bond prices must be positive")
    return (b[:-1] - b[1:]) / (accrual * b[1:])


# ---------------------------------------------------------------- LIBOR
LIBOR_STEPS = (10, 20, 40, 80)  # register-resident path kernels
# others: forward rates in shared memory up to 160 steps, in a per-CTA slice
# of global memory beyond (the reference takes any count, models.py:172-193;
# the cap is the Halton dimension cap, every base below 2^16)
LIBOR_MAX_STEPS = 6542


@dataclass(frozen=True)
class LiborConfig:
    """Caplet setup (models.py:172-193)."""

    valuation_time: float = 0.0
    maturity: float = 5.0
    accrual: float = 0.5
    strike: float = 0.01
    sigma: float = 0.04

    def __post_init__(self):
        if not 0 <= self.valuation_time < self.maturity:
            raise ValueError("need 0 <= valuation time < maturity")
        if self.accrual <= 0 or self.strike <= 0 or self.sigma < 0:
            raise ValueError("accrual and strike must be positive, sigma >= 0")
        if abs(self.maturity / self.accrual - round(self.maturity / self.accrual)) > 1e-9:
            raise ValueError("maturity must be an integer number of accrual periods")

    @property
    def steps(self) -> int:
        return round(self.maturity / self.accrual)


def black_caplet(config: LiborConfig, forward: float, bond: float,
                 sigma_prefactor: bool = False) -> float:
    """Black caplet price (models.py:249-268)."""
    if forward <= 0 or config.strike <= 0:
        raise ValueError("forward and strike must be positive")
    tau = config.maturity - config.valuation_time
    lead = config.sigma if sigma_prefactor else config.accrual
    if config.sigma == 0 or tau == 0:
        return lead * bond * max(forward - config.strike, 0.0)
    vol = config.sigma * math.sqrt(tau)
    d1 = (math.log(forward / config.strike) + 0.5 * vol * vol) / vol
    d2 = d1 - vol
    return lead * bond * (forward * norm_cdf(d1) - config.strike * norm_cdf(d2))


class LiborModel:
    """One-factor LIBOR market-model caplet (models.py:296-329)."""

    name = "libor"

    def __init__(self, config: LiborConfig | None = None, curve: YieldCurve | None = None):
        self.config = config or LiborConfig()
        self.curve = curve or default_curve()
        c = self.config
        bonds = bond_prices(self.curve, c.accrual, c.maturity + c.accrual)
        self.bonds = bonds
        self.initial_rates = init_libor(bonds, c.accrual)
        self.front_rate = (1.0 - bonds[0]) / (c.accrual * bonds[0])
        self.dim = c.steps
        if not 1 <= self.dim <= LIBOR_MAX_STEPS:
            raise ValueError(f"LIBOR steps {self.dim} outside 1..{LIBOR_MAX_STEPS}")

    def payoffs(self, u):
        """Discounted caplet payoffs for uniforms u[n, steps] (device kernel)."""
        return _payoffs(self, u)

    def black_price(self, sigma_prefactor: bool = False) -> float:
        return black_caplet(self.config, float(self.initial_rates[-1]), float(self.bonds[-1]),
                            sigma_prefactor)


# ---------------------------------------------------------------- MBS
@dataclass(frozen=True)
class MbsConfig:
    """Prepayment-model constants (models.py:337-370)."""

    initial_rate: float = 0.007
    k1: float = 0.01
    k2: float = -0.005
    k3: float = 10.0
    k4: float = 0.5
    variance: float = 0.0004
    months: int = 360
    payment: float = 1.0

    def __post_init__(self):
        if self.initial_rate <= 0:
            raise ValueError("initial_rate must be positive")
        if self.variance < 0:
            raise ValueError("variance must be >= 0")
        if self.months < 1:
            raise ValueError("months must be >= 1")

    @property
    def k0(self) -> float:
        return math.exp(-self.variance / 2.0)

    @property
    def sigma_xi(self) -> float:
        return math.sqrt(self.variance)

    def annuity_ratios(self) -> np.ndarray:
        """c_k = sum_{j=0}^{months-k} (1 + i0)^-j (models.py:366-370)."""
        j = np.arange(self.months, dtype=np.float64)
        return np.cumsum((1.0 + self.initial_rate) ** -j)[::-1].copy()


class MbsModel:
    """MBS present value (models.py:452-469)."""

    name = "mbs"

    def __init__(self, config: MbsConfig | None = None):
        self.config = config or MbsConfig()
        self.dim = self.config.months
        self.annuity = self.config.annuity_ratios()

    def payoffs(self, u):
        return _payoffs(self, u)


# ---------------------------------------------------------------- test integrands
class ConstantModel:
    """f(x) = 1 (models.py:477-486)."""

    name = "const1"

    def __init__(self, dim: int = 2):
        self.dim = dim

    def payoffs(self, u):
        return np.ones(np.shape(u)[0])


class FirstCoordinateModel:
    """f(x) = x_1, integral 1/2 (models.py:489-498)."""

    name = "x1"

    def __init__(self, dim: int = 2):
        self.dim = dim

    def payoffs(self, u):
        return np.array(u[:, 0], dtype=np.float64, copy=True)


class CoordinateHashModel:
    """Test integrand with no reference counterpart: payoff = the top 20
    bits of a 64-bit hash of every coordinate's bit pattern, in dimension
    order (include/rqmc_b200.h RQ_MODEL_XHASH).  Sums of such payoffs are
    exact, so theta pins all coordinates of all paths bit for bit where
    x1 only pins dimension 0."""

    name = "xhash"
    INIT = 0x6A09E667F3BCC909
    MUL = 0x9E3779B97F4A7C15

    def __init__(self, dim: int = 20):
        self.dim = dim

    def payoffs(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        bits = u.view(np.uint64)
        h = np.full(u.shape[0], self.INIT, dtype=np.uint64)
        with np.errstate(over="ignore"):
            for d in range(u.shape[1]):
                h = (h ^ bits[:, d]) * np.uint64(self.MUL)
                h ^= h >> np.uint64(32)
        return (h >> np.uint64(44)).astype(np.float64)


def _payoffs(model, u):
    torch = _lib.require_cuda()
    t, host = _as_device(u)
    if t.ndim != 2 or t.shape[1] != model.dim:
        raise ValueError(f"need uniforms of shape (n, {model.dim})")
    out = torch.empty(t.shape[0], dtype=torch.float64, device="cuda")
    st, keep = _lib.model_struct(model)
    _lib.check(_lib.lib().rq_model_payoffs(st, t.data_ptr(), t.shape[0], out.data_ptr(),
                                            _lib.stream_ptr()))
    torch.cuda.current_stream().synchronize()
    del keep
    return out.cpu().numpy() if host else out
