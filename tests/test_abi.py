"""The C-ABI library builds for sm_100a, loads here (no GPU), exports every
symbol include/mrq.h declares, and fails loudly without a device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mrq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mrq_[a-z_]+)\s*\(", src)))


def test_library_exports_all_declared_symbols():
    from paper_2411_06158_b200 import _build
    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    names = _declared()
    assert {"mrq_index_load", "mrq_search_batch", "mrq_free"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n


def test_sm100a_sass_present():
    import subprocess
    from paper_2411_06158_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2411_06158_b200 as m
    with pytest.raises(m.MRQError) as e:
        m.mrq_index_load(os.path.join(ROOT, "data", "tiny", "build_d16.mrqb"), np.zeros((10000, 64), np.float32), 16)
    assert e.value.code in (-6, -7)


def test_product_never_imports_oracle():
    """The product package and bench.py's main leg do not import oracle/."""
    pkg = os.path.join(ROOT, "paper_2411_06158_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
                assert "mrq_oracle" not in s and "liboracle" not in s, f
