#!/bin/bash
# One gpurun round trip: GPU tests, smoke, bench (plain runs only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
eval timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc $?"
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc $?"
fi
tail -25 gpurun_out/pytest_gpu.log
tail -3 gpurun_out/smoke.log
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
