cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_shards_check.log 2>&1
timeout 600 python scripts/c3_shards.py > gpurun_out/shards_check.log 2>&1
