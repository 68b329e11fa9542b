#!/bin/bash
# ncu evidence on the Deep-shaped search (the bench's operating point, np = 16,
# LOOSE) through scripts/probe_diag.py: the launch list of its searches and
# one --set full capture of each kernel of the second search.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CFG=${CFG:-deep}
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python scripts/probe_diag.py $CFG 16 > gpurun_out/launch_$CFG.log 2>&1
echo "launch list rc $?"
RX='k_rowmat|k_qtail|k_qorder|k_probe_tc|k_probe_finish|k_quant_g|k_cand_count|k_exclusive_scan|k_offsets_order|k_seed_w|k_scan|k_head|k_topk|k_stage2'
ncu --profile-from-start off --set full --clock-control none -k "regex:$RX" -s ${SKIP:-11} -c ${COUNT:-11} \
    -o gpurun_out/full_$CFG python scripts/probe_diag.py $CFG 16 > gpurun_out/full_$CFG.log 2>&1
echo "full rc $?"
tail -2 gpurun_out/full_$CFG.log
