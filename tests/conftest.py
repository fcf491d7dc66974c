import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu under gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle, build

    build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Ref()


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def unpack_blocks(g, prefix, L):
    """(idx, values, norm, size) per layer, or None for absent layers."""
    out = []
    for l in range(L):
        if f"{prefix}_absent_{l}" in g:
            out.append(None)
        else:
            out.append((g[f"{prefix}_idx_{l}"], g[f"{prefix}_val_{l}"], float(g[f"{prefix}_norm_{l}"]),
                        int(g[f"{prefix}_size_{l}"])))
    return out


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
