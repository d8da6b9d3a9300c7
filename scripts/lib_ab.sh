# A/B of library builds (ab/<variant>.so via EBL_LIB) on the C1 and C3 bench lines, interleaved,
# after the parity tests of the current build.   VARIANTS="cur x" bash scripts/lib_ab.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_lib_ab.log 2>&1
for rep in 1 2; do
 for v in ${VARIANTS:-cur}; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  for c in ${CONFIGS:-C1 C3}; do
   timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d.get('e2e') or {}; print('$v $c', 'value %.4g' % d['value'], 'e2e %.4g' % (e.get('value') or 0), 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'])"
  done
 done
done > gpurun_out/lib_ab.log 2>&1
