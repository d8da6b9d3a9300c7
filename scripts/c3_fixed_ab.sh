# C3: fixed tile regions (112-row tiles, regions 128 x W, compile-time words per row and the fast
# decide pass) for W = 128 / 192 / 256 (EBL_FIXED_W) vs the 64 x 256 tiles (EBL_FIXED_REGION=0)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharded_gpu.py tests/test_parity_gpu.py -q -x -k "c3 or shard or quiet or tile" > gpurun_out/pytest_c3_fixed.log 2>&1
for rep in 1 2; do for v in "0 128" "1 128" "1 192" "1 256"; do set -- $v
  EBL_FIXED_REGION=$1 EBL_FIXED_W=$2 timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('fixed=$1 w=$2', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'])"
done; done > gpurun_out/c3_fixed_ab.log 2>&1
for w in 192 256; do EBL_FIXED_W=$w timeout 1500 python -m pytest tests/test_sharded_gpu.py -q -x -k "c3_4096" >> gpurun_out/pytest_c3_fixed.log 2>&1; done
