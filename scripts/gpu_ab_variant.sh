# A/B of compile-time variants on one box: VARIANTS="base cb4" (base = libmrq.so), CFGS="deep sift"
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in ${CFGS:-deep sift}; do for v in ${VARIANTS:-base}; do
if [ "$v" = base ]; then unset MRQ_LIB_VARIANT; else export MRQ_LIB_VARIANT=$v; fi
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/abv_${cfg}_$v.json 2> gpurun_out/abv_${cfg}_$v.err
python3 -c "
import json; d=json.load(open('gpurun_out/abv_${cfg}_$v.json'))
print('$cfg $v value %.0f ms %.4f e2e %.0f recall %.4f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['recall10']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/abv_${cfg}_$v.err
done; done
