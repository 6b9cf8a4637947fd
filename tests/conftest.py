import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
TABLE = GOLDEN / "synthetic_11band.tbc"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhx.so")


def golden(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def words_to_int(words):
    return sum(int(w) << (64 * i) for i, w in enumerate(np.asarray(words, dtype=np.uint64)))


@pytest.fixture(scope="session")
def graphene_grid():
    return (-6.580201874549387, 14.863393148450246, 201)
