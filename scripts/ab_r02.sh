cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in cur micro pf1 micro_pf1 cur micro pf1 micro_pf1; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python scripts/c1_tail.py $v
done > gpurun_out/ab1.log 2>&1
unset EBL_LIB
TAIL_PROBE=1 python scripts/c1_tail.py cur >> gpurun_out/ab1.log 2>&1
EBL_LIB=$PWD/ab/prof.so python scripts/phase_warp.py prof > gpurun_out/phase_r02.log 2>&1
EBL_LIB=$PWD/ab/prof_pf1.so python scripts/phase_warp.py prof_pf1 >> gpurun_out/phase_r02.log 2>&1
python -m pytest tests -q -m gpu -k "c3_4096 or all_256 or learner or dem_nodata or wind_schedule or bench_c1_workload or side_configs" > gpurun_out/pytest_new_r02.log 2>&1
