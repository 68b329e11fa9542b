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


# ------------------------------------------------------ error paths (no GPU)
# mrq_index_load validates its arguments and the build file before any
# device work (include/mrq.h), so every error kind is testable on the CPU.

def _tiny_file(tmp_path):
    import synth
    from oracle import build as B
    cfg = synth.config_by_name("tiny")
    X, _ = synth.generate(cfg)
    src = os.path.join(ROOT, "data", "tiny", "build_d16.mrqb")
    raw = open(src, "rb").read()
    return X, raw, B.read(src)


def _load_err(path, X, d, **kw):
    import paper_2411_06158_b200 as m
    with pytest.raises(m.MRQError) as e:
        m.mrq_index_load(str(path), X, d, **kw)
    return e.value.code, str(e.value)


def test_load_error_kinds(tmp_path):
    """EIO, EVERSION, EFORMAT, EDIM, EINVAL."""
    import struct
    X, raw, bf = _tiny_file(tmp_path)
    p = tmp_path / "f.mrqb"
    # EIO: no such file
    assert _load_err(tmp_path / "missing.mrqb", X, 16)[0] == -9
    # EVERSION: bad magic, bad version
    p.write_bytes(b"XXXXXXXX" + raw[8:])
    assert _load_err(p, X, 16)[0] == -4
    p.write_bytes(raw[:8] + struct.pack("<I", 2) + raw[12:])
    assert _load_err(p, X, 16)[0] == -4
    p.write_bytes(raw[:5])                                          # shorter than the magic
    assert _load_err(p, X, 16)[0] == -4
    # EFORMAT: truncated header, header out of range, truncated payload, bad end marker, assignment >= k
    p.write_bytes(raw[:60])
    code, msg = _load_err(p, X, 16)
    assert code == -3 and "offset" in msg
    p.write_bytes(raw[:12] + struct.pack("<I", 0) + raw[16:])    # D = 0
    assert _load_err(p, X, 16)[0] == -3
    for cut in (200, len(raw) - 8 - 4 * 777, len(raw) - 3):
        p.write_bytes(raw[:cut])
        code, msg = _load_err(p, X, 16)
        assert code == -3 and "truncated at offset" in msg, (cut, msg)
    p.write_bytes(raw[:-8] + b"MRQEND02")
    code, msg = _load_err(p, X, 16)
    assert code == -3 and "end marker" in msg
    off = len(raw) - 8 - 4 * bf.N + 4 * 123                         # assignment of vector 123
    p.write_bytes(raw[:off] + struct.pack("<I", bf.k) + raw[off + 4:])
    code, msg = _load_err(p, X, 16)
    assert code == -3 and "vector 123" in msg
    # EDIM: D or d differ from the file's
    p.write_bytes(raw)
    assert _load_err(p, X[:, :32], 16)[0] == -2
    assert _load_err(p, X, 8)[0] == -2
    # EINVAL: n != N, d < 2, d > D
    assert _load_err(p, X[:-1], 16)[0] == -1
    assert _load_err(p, X, 1)[0] == -1
    assert _load_err(p, X, 65)[0] == -1


def test_huge_header_sizes_do_not_wrap(tmp_path):
    """Hostile header sizes (N = 2^32, k = 2^24) are rejected as EFORMAT/EINVAL
    before any size-dependent allocation (ADVICE: overflow-safe parsing)."""
    import struct
    X, raw, bf = _tiny_file(tmp_path)
    p = tmp_path / "h.mrqb"
    p.write_bytes(raw[:24] + struct.pack("<Q", 1 << 40) + raw[32:])
    assert _load_err(p, X, 16)[0] == -3
    p.write_bytes(raw[:20] + struct.pack("<I", 1 << 24) + raw[24:])   # k huge: payload far longer than the file
    assert _load_err(p, X, 16)[0] == -3


def test_python_binding_rejects_bad_shapes():
    """mrq.py checks query width and output buffers before calling the C ABI."""
    import paper_2411_06158_b200 as m
    import inspect
    src = inspect.getsource(m.mrq_search_batch) + inspect.getsource(m.mrq_search_batch_device)
    assert "MRQ_EDIM" in src and "_check_dev" in src
