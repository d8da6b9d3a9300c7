# C1 hand-over to the wide kernel: parity subset + A/B of EBL_BAIL / EBL_BAIL_AT; C3 prefetch variants
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pytest_bail.log 2>&1
for cfg in "1 0" "0 0" "1 60" "1 80" "1 120" "1 140"; do
  set -- $cfg
  EBL_BAIL=$1 EBL_BAIL_AT=$2 python scripts/c1_tail.py "bail=$1,at=$2"
done > gpurun_out/bail_ab.log 2>&1
for v in cur pf1 pf2; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],3), 'ms')"
done > gpurun_out/c3_pf.log 2>&1
unset EBL_LIB
for b in 1 0; do EBL_BAIL=$b python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bail=$b', 'value', round(d['value']/1e12,3), 'e2e', round(d['e2e']['value']/1e12,3), 'kern', round(d['roofline']['kernel_ms'],4))"; done >> gpurun_out/bail_ab.log 2>&1
