#!/bin/bash
# ncu --set full of one kernel (regex $1) in the probe_diag workload -> gpurun_out/$2.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:$1" -s ${SKIP:-1} -c 1 -o gpurun_out/$2 \
    python scripts/probe_diag.py ${CFG:-deep} ${NP:-16} > gpurun_out/$2.log 2>&1
tail -2 gpurun_out/$2.log
