# C3 tile geometry sweep (EBL_TILE_H x EBL_TILE_W; fixed regions with the compile-time fast pass)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
for th in ${THS:-16 24 32 40}; do for tw in ${TWS:-128 64}; do
  EBL_TILE_H=$th EBL_TILE_W=$tw timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('tile $th x $tw', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'])"
done; done; done > gpurun_out/c3_tiles.log 2>&1
