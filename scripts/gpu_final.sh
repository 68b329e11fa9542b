cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check.log 2>&1; grep "rc " gpurun_out/check.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config sift --steps 10 --warmup 3 > gpurun_out/bench_sift.json 2> gpurun_out/bench_sift.err; echo "sift rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"; cat gpurun_out/bench_ref.json | head -c 600
bash scripts/gpu_prof_sum.sh > gpurun_out/prof_sum.log 2>&1; tail -30 gpurun_out/prof_sum.log
