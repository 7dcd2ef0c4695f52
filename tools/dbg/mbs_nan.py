import sys; sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1408_5526_b200 import models as M
from paper_1408_5526_b200.harness import estimate_replications
SEED = 20120224
for var in [0.0004, 0.01, 0.02, 0.03, 0.04, 0.25]:
    m = M.MbsModel(M.MbsConfig(variance=var))
    for gen in ("philox", "rasrap-recursive"):
        try:
            th = estimate_replications(gen, m, SEED, 1, 4, (1000, 4096))
            print(var, gen, th[:, 1])
        except Exception as e:
            print(var, gen, "ERR", e)
    key = O.derive_key(SEED, 3, 1)
    w = O.philox_words(key, np.arange(4096), 360)
    u = w * 2.0**-32 + 2.0**-33
    ref = O.mbs_payoffs(u, m.config.initial_rate, m.config.k0, m.config.k1, m.config.k2, m.config.k3, m.config.k4, m.config.sigma_xi, m.config.payment, m.annuity)
    got = m.payoffs(u)
    bad = ~np.isfinite(got)
    print("payoffs_u: nonfinite", bad.sum(), "max rel", np.nanmax(np.abs(got/ref-1)))
    if bad.any():
        i = np.where(bad)[0][0]
        z = O.inv_normal(u[i])
        print(" path", i, "ref", ref[i], "z range", z.min(), z.max())
        # month at which it goes bad: payoffs of truncated models
        for mo in (20, 60, 120, 180, 240, 300, 360):
            mm = M.MbsModel(M.MbsConfig(variance=var, months=mo))
            print("  months", mo, mm.payoffs(u[i:i+1, :mo]))
