"""The product path has no CPU fallback: without the library or without a
CUDA device every device entry point raises (CPU tests)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, SEED


def test_missing_library_raises_importerror(tmp_path):
    code = ("from paper_1408_5526_b200 import _lib\n"
            "try:\n    _lib.lib()\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n")
    env = dict(os.environ, RQMC_B200_LIB=str(tmp_path / "nope.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert "IMPORTERROR" in out.stdout and "no CPU fallback" in out.stdout


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_device_entry_points_raise_without_cuda():
    import paper_1408_5526_b200 as P
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200._lib import DeviceError

    with pytest.raises(DeviceError):
        P.make_sampler("rasrap-recursive", 20, SEED, 1).fill(np.empty((8, 20)))
    model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    with pytest.raises(DeviceError):
        model.payoffs(np.full((4, model.dim), 0.5))
    cfg = P.ExperimentConfig(model="libor", generator="philox", n_grid=(128,), replications=2,
                             seed=SEED)
    with pytest.raises(DeviceError):
        P.run_experiment(cfg, model=model)
