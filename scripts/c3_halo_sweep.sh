# C3: light-cone halo rows = steps per launch (EBL_TILE_HALO) x tile height, 128-column tiles
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out

for rep in 1 2; do for v in "16 32" "20 32" "24 32" "32 32" "16 24" "16 16" "24 24" "24 16"; do set -- $v
  EBL_TILE_HALO=$1 EBL_TILE_H=$2 EBL_TILE_W=128 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('halo $1 tile_h $2', 'ms %.4f' % d['ms_per_step'], 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'], 'launches', d['gpu_launches'])"
done; done > gpurun_out/c3_halo_sweep.log 2>&1
