cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_sharded_gpu.py tests/test_parity_gpu.py tests/test_synth_gpu.py tests/test_bench_contract.py -q -x > gpurun_out/pytest_halo16.log 2>&1
for rep in 1 2; do timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C3', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'], 'e2e %.4g' % d['e2e']['value'], 'launches', d['gpu_launches'])"; done > gpurun_out/halo16.log 2>&1
timeout 600 python scripts/c3_shards.py >> gpurun_out/halo16.log 2>&1
