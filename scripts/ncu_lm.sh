cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_scan_tc|k_lm_" -s 4 -c 4 \
    -o gpurun_out/full_lm python scripts/probe_diag.py deep 16 > gpurun_out/full_lm.log 2>&1
echo "full rc $?"
