# C1 A/B of library builds: parity tests of the current build, then per variant the bench line and
# the critical-path probe (scripts/c1_tail.py), interleaved.   VARIANTS="cur x" bash scripts/c1_ab.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_synth_gpu.py -q -x > gpurun_out/pytest_c1_ab.log 2>&1
for rep in 1 2; do
 for v in ${VARIANTS:-cur}; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v bench', 'value %.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], 'kern %.4f' % d['roofline']['kernel_ms'])"
  timeout 600 python scripts/c1_tail.py $v
 done
done > gpurun_out/c1_ab.log 2>&1
