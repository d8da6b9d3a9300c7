# C3 geometry sweep: light-cone halo rows (= steps per launch, EBL_TILE_HALO) x tile height x width
#   VS="16_32_128 8_32_128" bash scripts/c3_halo_sweep.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do for v in ${VS:-4_32_128 8_32_128 12_32_128 16_32_128 24_32_128 16_32_64 16_32_256 16_48_128}; do
  set -- $(echo $v | tr _ ' ')
  EBL_TILE_HALO=$1 EBL_TILE_H=$2 EBL_TILE_W=$3 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('halo $1 tile $2 x $3', 'kern %.4f' % d['roofline']['kernel_ms'], 'tiles %.4f' % d['tiles_processed_frac'])"
done; done > gpurun_out/c3_halo_sweep.log 2>&1
