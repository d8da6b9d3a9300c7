# C3 tile geometry sweep (EBL_TILE_H x EBL_TILE_W) with the work-list launches, + tanker per-step A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for th in 64 112 56; do for tw in 256 128 64; do
  EBL_TILE_H=$th EBL_TILE_W=$tw python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('tile $th x $tw', round(d['ms_per_step'],3), 'ms', 'tiles', round(d['tiles_processed_frac'],4), 'launches', d['gpu_launches'])"
done; done > gpurun_out/c3_tiles.log 2>&1
VARIANTS="cur rlnofast" bash scripts/c2_ab.sh
