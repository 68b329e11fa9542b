#!/bin/bash
# bench only (plain run) + the stage times; optional ncu launch list of probe_diag (LAUNCHES=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc $?"
python3 -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.0f ms %.4f e2e %.0f' % (d['value'], d['ms_per_step'], d['e2e']['value']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/bench.err
if [ -n "$LAUNCHES" ]; then
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${CFG:-deep}.csv python scripts/probe_diag.py ${CFG:-deep} 16 > /dev/null 2>&1
  python3 scripts/launch_table.py gpurun_out/launches_${CFG:-deep}.csv
fi
