cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:${KRX:-k_scan|k_head_topk}" -s ${SKIP:-2} -c ${COUNT:-2} \
    -o gpurun_out/full_hot python scripts/probe_diag.py deep 16 > gpurun_out/full_hot.log 2>&1
echo "full rc $?"
tail -3 gpurun_out/full_hot.log
ls -la gpurun_out/full_hot.ncu-rep
