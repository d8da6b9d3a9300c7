cd /root/repo
python scripts/one_env_copies.py heaviest 148 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 3 -c 1 -o gpurun_out/prof_heavy148 python scripts/one_env_copies.py heaviest 148 > gpurun_out/ncu_heavy.log 2>&1
echo rc=$?
