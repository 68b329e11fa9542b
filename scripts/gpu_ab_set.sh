# A/B of mrq_debug_set switches on one box: SETS="quant_split=0 quant_split=1", CFGS="deep sift"
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
if [ -n "$KEXPR" ]; then timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -m gpu -q -x -k "$KEXPR" > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/quick_pytest.log; fi
for cfg in ${CFGS:-deep sift}; do for v in ${SETS}; do
MRQ_DEBUG_SET=$v timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/abs_${cfg}_$v.json 2> gpurun_out/abs_${cfg}_$v.err
python3 -c "
import json; d=json.load(open('gpurun_out/abs_${cfg}_$v.json'))
print('$cfg $v value %.0f ms %.4f e2e %.0f recall %.4f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['recall10']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/abs_${cfg}_$v.err
done; done
