# C2 A/B of library variants (bench C2 env-steps/s) + the RL parity tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_rl_gpu.py -q -x > gpurun_out/pytest_rl_r02.log 2>&1
for v in ${VARIANTS:-cur rllut}; do
 for rep in 1 2; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M env-steps/s', 'e2e', round(d['e2e']['value']/1e6,2), 'device_io', round(d['device_io_step']['env_steps_per_sec']/1e6,1))"
 done
done > gpurun_out/c2_ab.log 2>&1
