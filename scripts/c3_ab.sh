# C3 work-list launches vs grid launches (EBL_WORK_LIST), bench C3 + the parity tests of tiled runs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py tests/test_sharded_gpu.py tests/test_synth_gpu.py -q -x > gpurun_out/pytest_c3_r02.log 2>&1
for wl in 1 0 1 0; do
  EBL_WORK_LIST=$wl python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('worklist=$wl', round(d['ms_per_step'],3), 'ms', round(d['value']/1e12,2), 'e12', 'tiles', d['tiles_processed_frac'], 'launches', d['gpu_launches'])"
done > gpurun_out/c3_ab.log 2>&1
