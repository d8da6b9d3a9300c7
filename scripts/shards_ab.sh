# Row-shard checks: sharded tests, then C3 16384^2 x 500 as G = 1/2/4/8 fused shards on one GPU
# (+ the per-rank form's tile share) with and without the tile-record exchange (EBL_HALO_MARKS).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_shards_marks.log 2>&1
timeout 600 python scripts/c3_shards.py > gpurun_out/c3_shards_marks.log 2>&1
EBL_HALO_MARKS=0 timeout 600 python scripts/c3_shards.py 16384 500 8 > gpurun_out/c3_shards_nomarks.log 2>&1
