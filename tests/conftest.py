import glob
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running checks")


def golden_cases():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def oracle_params(g):
    from oracle.fvm_oracle import Params
    soc, i00pl = g["params"]
    return Params(soc_init=float(soc), i00_plel=float(i00pl))


def scaled_err(a, b, scale):
    """max_i |a_i - b_i| / max(scale_i, tiny): relative agreement per row."""
    scale = np.maximum(np.abs(scale), 1e-300)
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / scale)) if np.size(a) else 0.0
