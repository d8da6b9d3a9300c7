# C3: k_tile_init (records + first list, no grid launch; default) vs the grid first launch
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharded_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_tile_init.log 2>&1
for rep in 1; do for x in 1; do
  EBL_TILE_INIT=$x timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('init=$x', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'], 'launches', d['gpu_launches'])"
done; done > gpurun_out/tile_init_ab.log 2>&1
