# Programmatic dependent launch (default) vs plain launches (ab/nopdl.so): C3, shards, C4 + tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharded_gpu.py tests/test_det_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_pdl.log 2>&1
for rep in 1 2; do for v in cur nopdl; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  for c in C3 C4; do
   timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $c', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'])"
  done
  C3_REPS=3 C3_PER_RANK=0 timeout 600 python scripts/c3_shards.py 16384 500 8 | sed "s/^/$v /"
done; done > gpurun_out/pdl_ab.log 2>&1
