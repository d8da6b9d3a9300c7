cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_resident -s 3 -c 1 -o gpurun_out/prof_resident $CMD > gpurun_out/ncu_full.log 2>&1
CMDT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --kernel tiled"
$CMDT > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_tile -s 700 -c 1 -o gpurun_out/prof_tile $CMDT > gpurun_out/ncu_full_tile.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
