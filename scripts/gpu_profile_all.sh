# Final evidence run (under gpurun from the repo root): bench line, all-config lines, the C1 launch
# list + full capture, C2, C3 and C4 captures (each profiled command first runs plain, && ncu).
cd "${GRAFT_REPO_ROOT:-.}"
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.log 2>&1
python scripts/bench_configs.py --configs c0,c2,c3,c4 --iters 5 > gpurun_out/configs_final.jsonl 2> gpurun_out/configs_final.err
C1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$C1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $C1 > gpurun_out/ncu_launches_c1.log 2>&1
$C1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 3 -c 1 -o gpurun_out/prof_c1 $C1 > gpurun_out/ncu_c1.log 2>&1
C2="python scripts/bench_configs.py --configs c2 --iters 1"
$C2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_rl_tanker_warp -s 3 -c 1 -o gpurun_out/prof_c2 $C2 > gpurun_out/ncu_c2.log 2>&1
C3="python scripts/bench_configs.py --configs c3 --iters 1 --c3-size 4096"
$C3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 70 -c 1 -o gpurun_out/prof_c3 $C3 > gpurun_out/ncu_c3.log 2>&1
C4="python scripts/bench_configs.py --configs c4 --iters 1"
$C4 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $C4 > gpurun_out/ncu_launches_c4.log 2>&1
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_back -s 50 -c 1 -o gpurun_out/prof_c4back $C4 > gpurun_out/ncu_c4back.log 2>&1
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_forward -s 50 -c 1 -o gpurun_out/prof_c4fwd $C4 > gpurun_out/ncu_c4fwd.log 2>&1
echo done
