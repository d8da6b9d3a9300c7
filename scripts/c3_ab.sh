# C3 A/B of library builds (ab/<variant>.so) + the sharded / parity tests of the current build
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharded_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_c3_ab.log 2>&1
for rep in 1 2; do for v in ${VARIANTS:-cur base}; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v C3', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'])"
  C3_REPS=3 C3_PER_RANK=0 timeout 600 python scripts/c3_shards.py 16384 500 8 | sed "s/^/$v /"
done; done > gpurun_out/c3_ab.log 2>&1
