# Our arm's bench lines of every config (after a counters refresh), TAG-named
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-r02}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}_default.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c1.log 2>&1
for c in C0 C2 C3 C4; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_${c,,}.log 2>&1
done
