"""Locate the installed reference package (baseline/_ref, built by the one allowed offline install; it
travels to the GPU box with the snapshot) for the drop-in tests.  Tests that need it skip without it."""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_SITE = ROOT / "baseline" / "_ref"


def import_hexmc():
    if not (REF_SITE / "hexmc").is_dir():
        pytest.skip("reference package not installed under baseline/_ref")
    os.environ.setdefault("HEXMC_NO_NUMBA", "1")  # the reference's pure-numpy kernels (_kernels.py:19-29)
    if str(REF_SITE) not in sys.path:
        sys.path.insert(0, str(REF_SITE))
    import hexmc.cli
    import hexmc.config
    import hexmc.runner

    return hexmc
