# ncu captures (run under gpurun from the repo root).  Each profiled command first runs plain
# (&&) so ncu only sees commands that exit 0 on their own.
cd "${GRAFT_REPO_ROOT:-.}"
C1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$C1 > gpurun_out/prof_c1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $C1 > gpurun_out/ncu_launches_c1.log 2>&1
$C1 > gpurun_out/prof_c1_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_blocked -s 3 -c 1 -o gpurun_out/prof_c1 $C1 > gpurun_out/ncu_c1.log 2>&1
C2="python scripts/bench_configs.py --configs c2 --iters 1"
$C2 > gpurun_out/prof_c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rl_tanker_bits -s 3 -c 1 -o gpurun_out/prof_c2 $C2 > gpurun_out/ncu_c2.log 2>&1
C3="python scripts/bench_configs.py --configs c3 --iters 1 --c3-size 4096"
$C3 > gpurun_out/prof_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_blocked -s 70 -c 1 -o gpurun_out/prof_c3 $C3 > gpurun_out/ncu_c3.log 2>&1
C4="python scripts/bench_configs.py --configs c4 --iters 1"
$C4 > gpurun_out/prof_c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $C4 > gpurun_out/ncu_launches_c4.log 2>&1
