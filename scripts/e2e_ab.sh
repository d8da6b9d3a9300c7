# C1 end to end: zero-copy input (one launch) vs the chunked copy pipeline
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -q -x -k "pipelined or bench_c1" > gpurun_out/pytest_e2e.log 2>&1
for z in 1 0 1 0; do EBL_PIPE_ZCIN=$z python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('zcin=$z', 'value', round(d['value']/1e12,3), 'e2e', round(d['e2e']['value']/1e12,3), 'e2e ms', round(d['e2e']['ms_per_step'],4), 'kern', round(d['roofline']['kernel_ms'],4))"; done > gpurun_out/e2e_ab.log 2>&1
