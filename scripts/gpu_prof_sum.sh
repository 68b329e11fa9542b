# ncu launch list + --set full capture of one search per config, summarised ON the box
# (the reports exceed gpurun's 64 MiB return limit): gpurun_out/{launches,ncu_full_summary,ncu_traffic}_<cfg>.*
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for CFG in ${CFGS:-deep sift}; do
  export CFG
  bash scripts/gpu_prof_deep.sh
  python scripts/ncu_summary.py gpurun_out/full_$CFG.ncu-rep gpurun_out/ncu_full_summary_$CFG.json --traffic gpurun_out/ncu_traffic_$CFG.json
  rm -f gpurun_out/full_$CFG.ncu-rep
done
