#!/bin/bash
# A/B build: copy the committed-or-working tree (sources only) to ./<name>/
# (git-ignored, travels with gpurun) and build it with extra nvcc flags.
# usage: scripts/variant.sh NAME "-DFOO=1 ..."   (data/ is shared via symlink)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
rm -rf "$name"; mkdir "$name"
tar --exclude=./data --exclude=./gpurun_out --exclude=./.git --exclude='./ab*' --exclude='./var_*' -cf - . | tar -xf - -C "$name"
ln -s ../data "$name/data"
rm -f "$name"/paper_2411_06158_b200/libmrq.so
(cd "$name" && MRQ_NVCC_EXTRA="$*" python -c "from paper_2411_06158_b200 import _build; _build.build(force=True)")
echo "built $name with: $*"
