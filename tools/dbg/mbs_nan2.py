import sys, math; sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1408_5526_b200 import models as M
SEED = 20120224
var = 0.04
key = O.derive_key(SEED, 3, 1)
w = O.philox_words(key, np.arange(473), 360)
u = (w * 2.0**-32 + 2.0**-33)[472:473]
z = O.inv_normal(u[0])
prev = None
for mo in range(1, 361):
    mm = M.MbsModel(M.MbsConfig(variance=var, months=mo))
    v = mm.payoffs(u[:, :mo])[0]
    if not np.isfinite(v):
        print("first nonfinite at months", mo, "prev", prev); break
    prev = v
# reference-style trace
c = M.MbsConfig(variance=var)
i = c.initial_rate; k0 = c.k0; sx = c.sigma_xi
for k in range(mo):
    i = k0 * math.exp(sx * z[k]) * i
print("z at", mo-1, z[mo-1], "rate", i, "y", c.k3 * i + c.k4)
for k in range(max(0, mo-6), mo):
    print(k, z[k])
