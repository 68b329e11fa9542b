# quick check of a scan / stage change: the sketch + stagewise parity tests, then the Deep- and SIFT-shaped bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${KEXPR:-sketch or stagewise or head_topk}" > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/quick_pytest.log
for cfg in ${CFGS:-deep sift}; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/quick_${cfg}.json 2> gpurun_out/quick_${cfg}.err
python3 -c "
import json; d=json.load(open('gpurun_out/quick_${cfg}.json'))
print('$cfg value %.0f ms %.4f e2e %.0f recall %.4f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['recall10']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/quick_${cfg}.err
done
