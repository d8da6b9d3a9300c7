# ncu evidence for the C1 bench kernel (run under gpurun from the repo root): the launch list of
# the bench command and one full capture of the dominant kernel, each after a plain run exits 0.
cd "${GRAFT_REPO_ROOT:-.}"
K=${K:-k_step_warp}
C1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$C1 > gpurun_out/prof_c1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $C1 > gpurun_out/ncu_launches_c1.log 2>&1
$C1 > gpurun_out/prof_c1_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_c1 $C1 > gpurun_out/ncu_c1.log 2>&1
echo done
