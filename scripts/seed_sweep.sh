#!/bin/bash
# Bench the decision-T seed-pool settings (GPU box).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "1 2" "2 2" "4 2" "2 4" "4 4" "8 4" "4 6"; do
  set -- $cfg
  python bench.py --steps 5 --warmup 3 --no-cpu --seed-lists $1 --seed-mult $2 > gpurun_out/seed_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/seed_$1_$2.json')); c=d['config']
print('seed_lists=$1 seed_mult=$2', d['value'], d['ms_per_step'], 'recall', c['recall10'], 'exact/q', c['exact_per_query'], c['stage_ms'])"
done
