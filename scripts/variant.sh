#!/bin/bash
# A/B build of a compile-time variant: builds libmrq_<name>.so next to
# libmrq.so with extra nvcc flags (objects are cached per flag set under
# paper_2411_06158_b200/build/).  Load it with MRQ_LIB_VARIANT=<name>.
# usage: scripts/variant.sh NAME "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/.."
name=$1; shift
MRQ_NVCC_EXTRA="$*" python - <<PY
import os, shutil
from paper_2411_06158_b200 import _build
lib = _build.LIB
tmp = lib + ".main"
if os.path.exists(lib):
    shutil.copy2(lib, tmp)
try:
    _build.LIB = lib.replace("libmrq.so", "libmrq_$name.so")
    _build.build(force="relink")
finally:
    if os.path.exists(tmp):
        os.replace(tmp, lib)
print("built", _build.LIB)
PY
