#!/bin/bash
# ncu evidence: launch list of one bench invocation + full sets of the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1
rc=$?
echo "plain rc $rc"
if [ $rc -ne 0 ]; then tail -20 gpurun_out/plain.log; exit 1; fi
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc $?"
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_stage2_w|k_scan|k_probe_select_w|k_probe_approx|k_seed_w}" -s ${SKIP:-25} -c ${COUNT:-5} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc $?"
tail -3 gpurun_out/ncu_full.log
