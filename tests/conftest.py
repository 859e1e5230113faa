import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "golden.json").read_text())
    arrays = dict(np.load(GOLDEN / "golden.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True

# the staged reference suite runs only through tests/test_ref_compat.py (moesim alias)
collect_ignore_glob = ["ref_compat/*"]


def pytest_terminal_summary(terminalreporter):
    """Near-tie report (never silently): every selection
    comparison against the oracle that tolerated a near-tie order flip."""
    from tests.helpers import NEAR_TIES
    if not NEAR_TIES:
        return
    ties = [t for t in NEAR_TIES if t[2]]
    terminalreporter.write_line(
        f"[near-ties] {sum(t[2] for t in NEAR_TIES)} near-tie layer(s) in {len(ties)} of {len(NEAR_TIES)} "
        f"selection comparisons ({sum(t[1] for t in NEAR_TIES)} layers compared); per comparison <= "
        f"{__import__('tests.helpers', fromlist=['MAX_NEAR_TIES']).MAX_NEAR_TIES}")
    for tid, n, k in ties[:20]:
        terminalreporter.write_line(f"[near-ties]   {tid}: {k} of {n} layers")
