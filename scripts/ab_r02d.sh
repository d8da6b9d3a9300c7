cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python scripts/c1_tail.py cur > gpurun_out/ab4.log 2>&1
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C3', round(d['ms_per_step'],3), 'ms', d['gpu_launches'])" >> gpurun_out/ab4.log 2>&1
VARIANTS="cur" bash scripts/c2_ab.sh
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_r02d.log 2>&1
