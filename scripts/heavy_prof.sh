cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python scripts/one_env_copies.py heaviest 148 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 2 -c 1 -o gpurun_out/prof_r02_heavy148 python scripts/one_env_copies.py heaviest 148 > gpurun_out/ncu_heavy.log 2>&1
python scripts/one_env_copies.py median 148 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 2 -c 1 -o gpurun_out/prof_r02_median148 python scripts/one_env_copies.py median 148 > gpurun_out/ncu_median.log 2>&1
