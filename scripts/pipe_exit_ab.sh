# C1 e2e: the pipeline's launches with (EBL_PIPE_EXIT=1) and without the early-exit instantiation
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
EBL_PIPE_EXIT=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "pipelined or bench_c1" > gpurun_out/pytest_pipe_exit.log 2>&1
for rep in 1 2 3; do for x in 0 1; do
  EBL_PIPE_EXIT=$x timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('exit=$x', 'value %.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], 'e2e_ms %.4f' % d['e2e']['ms_per_step'])"
done; done > gpurun_out/pipe_exit_ab.log 2>&1
