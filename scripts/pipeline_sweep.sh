# C1 e2e: chunk count of the host-buffer pipeline (ebl_batch_set_pipeline) x zero-copy output chunks
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
 for p in 2 3 4 6 8; do
  for zc in -1 0; do
   EBL_PIPE_ZC=$zc timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline $p 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chunks=$p zc=$zc', 'e2e %.4g' % d['e2e']['value'], 'e2e_ms %.4f' % d['e2e']['ms_per_step'])"
  done
 done
done > gpurun_out/pipeline_sweep.log 2>&1
