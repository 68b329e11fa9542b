cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in ${CFGS:-deep}; do for g in ${GROUPS_:-128 256 512 1024 2048}; do
MRQ_QO_GROUPS=$g timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_${cfg}_g$g.json 2> gpurun_out/ab_${cfg}_g$g.err
python3 -c "
import json; d=json.load(open('gpurun_out/ab_${cfg}_g$g.json'))
print('$cfg groups=$g value %.0f ms %.4f e2e %.0f load %.2f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['index_load_s']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/ab_${cfg}_g$g.err
done; done
