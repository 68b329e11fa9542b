cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_scan|k_head_topk|k_seed_w|k_probe_tc|k_quant_g" -s 5 -c 5 \
    -o gpurun_out/full_hot python scripts/probe_diag.py deep 16 > gpurun_out/full_hot.log 2>&1
echo "full rc $?"
tail -3 gpurun_out/full_hot.log
