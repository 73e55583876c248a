import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith(("scale_", "symbolic_")))


def mesh_of(g):
    import paper_2306_08994_b200 as tf
    dims = tuple(int(x) for x in g["dims"])
    p = int(g["degree"])
    return tf.TensorMesh(dims, p) if len(dims) > 1 else tf.Mesh(dims[0], p)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
