# C4 evidence of this build: the bench line, the per-launch DRAM bytes of one run (ncu metrics pass
# over the k_det_* launches -> profiles/ncu_counters.json "c4:..."), one full capture of the
# streaming backward.  Run under gpurun from the repo root.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline"
$C4 > gpurun_out/c4_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'k_det_(forward|back|loss|reduce|bd_run)' -c 220 --csv --log-file gpurun_out/c4_metrics.csv $C4 > gpurun_out/c4_ncu_metrics.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_det_back_stream -s 450 -c 1 \
    -o gpurun_out/prof_r02_c4stream $C4 > gpurun_out/ncu_c4stream.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_det_forward -s 450 -c 1 \
    -o gpurun_out/prof_r02_c4fwd $C4 > gpurun_out/ncu_c4fwd.log 2>&1
