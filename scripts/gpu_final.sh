# round-end check: GPU suite, smoke, the default bench line, the other shapes, the reference arm
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check.log 2>&1; grep "rc " gpurun_out/check.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config sift --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_sift.json 2> gpurun_out/bench_sift.err; echo "sift rc $?"
timeout 600 python bench.py --config gist --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_gist.json 2> gpurun_out/bench_gist.err; echo "gist rc $?"
timeout 600 python bench.py --config deep --K 100 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_deep_k100.json 2> gpurun_out/bench_deep_k100.err; echo "k100 rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
for f in bench bench_sift bench_gist bench_deep_k100; do python3 -c "
import json; d=json.load(open('gpurun_out/$f.json'))
print('$f', d['config']['workload'][:12], 'value %.0f ms %.4f e2e %.0f recall %.4f np %d %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['recall10'], d['config']['nprobe'], d['config']['tau_schedule']))
"; done
