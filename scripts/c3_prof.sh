# C3 launch list + a full capture of a mid-run work-list launch, + bench C3 and the tanker A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
C3="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline"
$C3 > gpurun_out/c3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $C3 > /dev/null 2>&1
$C3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 290 -c 1 -o gpurun_out/prof_r02_c3list $C3 > gpurun_out/ncu_c3.log 2>&1
python -m pytest tests/test_sharded_gpu.py tests/test_rl_gpu.py -q -x > gpurun_out/pytest_c3b.log 2>&1
VARIANTS="cur rlnofast" bash scripts/c2_ab.sh
