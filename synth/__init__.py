"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_2411_06158_b200/``).  It holds none of the method's arithmetic:
no PCA, no k-means, no quantizer, no distance estimator.  It only draws base
vectors and queries (BASELINE.json ``configs``).

The paper measures on eight public datasets (Table 1);
none is available here, so these generators stand in for them.  No dataset
item is reproduced.
"""
from .generator import generate, CONFIGS, Config, config_by_name, base_sha256  # noqa: F401
