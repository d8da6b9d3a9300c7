cd "${GRAFT_REPO_ROOT:-.}"
timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -k pipelined > gpurun_out/pipe_test.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_test.log
for c in 1 2 4 8 16 32 64; do
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline $c > gpurun_out/pipe_$c.log 2>&1
done
