# Launch lists (ncu, cold and serialised) of C3 16384^2 x 500: unsharded vs 8 fused shards on one GPU.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
C3_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shards_launches.csv \
  python scripts/c3_shards.py 16384 500 8 > gpurun_out/shards_ncu.log 2>&1
