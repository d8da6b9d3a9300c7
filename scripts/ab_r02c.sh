cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python scripts/c1_tail.py cur > gpurun_out/ab3.log 2>&1
python scripts/c1_tail.py cur >> gpurun_out/ab3.log 2>&1
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C3', round(d['ms_per_step'],3), 'ms', d['gpu_launches'])" >> gpurun_out/ab3.log 2>&1
VARIANTS="cur rlnofast rllut" bash scripts/c2_ab.sh
