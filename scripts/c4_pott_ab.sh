# C4 forward with the target-ordered pot table vs the source-ordered one (EBL_DET_POTT), + det tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_det_gpu.py -q -x > gpurun_out/pytest_det_pott.log 2>&1
for p in 1 0 1 0; do EBL_DET_POTT=$p python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('pott=$p', round(d['ms_per_step'],3), 'ms', 'cal', round(d['calibrate_ms_per_iteration'],2), 'loss', d['loss_sum'])"; done > gpurun_out/c4_pott.log 2>&1
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline"
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_forward -s 450 -c 1 -o gpurun_out/prof_r02_c4fwd_pott $C4 > /dev/null 2>&1
