#!/bin/bash
# list-major scan: parity subset, then bench A/B (lm on / off / variants)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 600 -k "list_major or head_sketch or stagewise or fused_equals" > gpurun_out/pytest_lm.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/pytest_lm.log
for v in ${VARIANTS:-"main:"}; do
  name=${v%%:*}; set=${v#*:}
  lib=""; [ "$name" != main ] && [ "${name#lib_}" != "$name" ] && lib=${name#lib_}
  MRQ_LIB_VARIANT=$lib MRQ_DEBUG_SET=$set timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_$name.json'))
print('$name', 'value %.0f ms %.4f recall %.4f' % (d['value'], d['ms_per_step'], d['config']['recall10']))
print({k: v for k, v in d['config']['stage_ms'].items() if v > 0.003})
" || tail -5 gpurun_out/bench_$name.err
done
