# One GPU round trip (run under gpurun from the repo root): parity tests, smoke, bench,
# then the ncu launch list + one full capture of the dominant kernel.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -v --tb=short --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
if [ "${PROFILE:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
  $CMD > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_step_blocked -s 3 -c 1 -o gpurun_out/prof_blocked $CMD > gpurun_out/ncu_full.log 2>&1
fi
