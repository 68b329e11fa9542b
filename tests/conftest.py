import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def tiny():
    """Tiny config (BASELINE.json configs[0]) with its oracle build + encode."""
    import numpy as np  # noqa: F401
    import synth
    import oracle
    from oracle import build as B
    cfg = synth.config_by_name("tiny")
    X, Q = synth.generate(cfg)
    bf = B.build(X, cfg.d[0], cfg.k)
    ix = oracle.Index(bf, X)
    return cfg, X, Q, bf, ix
