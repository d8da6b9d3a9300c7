# C2 per-step host-buffer path: zero-copy actions / reward / done (default) vs copies (EBL_RL_ZC=0)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rl_gpu.py -q -x > gpurun_out/pytest_rl_zc.log 2>&1
for rep in 1 2; do for z in 2 0; do
  EBL_RL_ZC=$z timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('zc=$z', 'value %.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], 'dio %.4g' % d['device_io_step']['env_steps_per_sec'])"
done; done > gpurun_out/c2_zc_ab.log 2>&1
