# A/B of the decision-T seed parameters on the Deep-shaped bench: SWEEP="lists:mult ..."
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for s in ${SWEEP:-2:2 2:3 2:4 3:3}; do
sl=${s%%:*}; sm=${s##*:}
timeout 600 python bench.py --config ${CFG:-deep} --steps 10 --warmup 3 --no-cpu --seed-lists $sl --seed-mult $sm > gpurun_out/sl_${sl}_$sm.json 2> gpurun_out/sl_${sl}_$sm.err
python3 -c "
import json; d=json.load(open('gpurun_out/sl_${sl}_$sm.json'))
print('seed_lists=$sl seed_mult=$sm value %.0f ms %.4f recall %.4f f1 %.1f surv %.1f exact %.1f' % (d['value'], d['ms_per_step'], d['config']['recall10'], d['config']['f1_per_query'], d['config']['sketch_pass_per_query'], d['config']['exact_per_query']))
print(d['config']['stage_ms'])
" || tail -5 gpurun_out/sl_${sl}_$sm.err
done
