# Evidence run (under gpurun from the repo root): the GPU suite + smoke, the bench lines of every
# config (ours + the reference arm), the C1 launch list + full capture of the dominant kernel,
# C2 / C4 captures, the C3 shard measurement.  Every profiled command first runs plain (&& ncu).
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
python bench.py > gpurun_out/bench_${TAG}_default.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c1_ref.log 2>&1
for c in C0 C2 C3 C4; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_${c,,}.log 2>&1
  python bench.py --config $c --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${TAG}_${c,,}_ref.log 2>&1
done
C1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$C1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c1.csv $C1 > gpurun_out/ncu_launches_c1.log 2>&1
$C1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 3 -c 1 -o gpurun_out/prof_${TAG}_c1 $C1 > gpurun_out/ncu_c1.log 2>&1
C2="python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline"
$C2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_rl_tanker_warp -s 3 -c 1 -o gpurun_out/prof_${TAG}_c2 $C2 > gpurun_out/ncu_c2.log 2>&1
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline"
$C4 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $C4 > gpurun_out/ncu_launches_c4.log 2>&1
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_back_stream -s 450 -c 1 -o gpurun_out/prof_${TAG}_c4back $C4 > gpurun_out/ncu_c4back.log 2>&1
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_forward -s 450 -c 1 -o gpurun_out/prof_${TAG}_c4fwd $C4 > gpurun_out/ncu_c4fwd.log 2>&1
C3="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline"
$C3 > /dev/null 2>&1 && ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_step_warp -c 40 --csv --log-file gpurun_out/c3_metrics_${TAG}.csv $C3 > gpurun_out/ncu_c3.log 2>&1
python scripts/c3_shards.py > gpurun_out/c3_shards_${TAG}.log 2>&1
echo done
