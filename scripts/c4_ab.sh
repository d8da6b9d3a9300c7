# C4 A/B of library variants (bench C4 ms/step) + det parity tests + ncu of the streaming backward
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m pytest tests/test_det_gpu.py -q -x > gpurun_out/pytest_det_r02.log 2>&1
for v in ${VARIANTS:-cur nostream}; do
 for rep in 1 2; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],3), 'ms', 'e2e', round(d['e2e']['value']/1e9,2), 'Gcs/s', 'loss', d['loss_sum'])"
 done
done > gpurun_out/c4_ab.log 2>&1
unset EBL_LIB
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline"
$C4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_det_back_stream -s 450 -c 1 -o gpurun_out/prof_r02_c4stream $C4 > gpurun_out/ncu_c4stream.log 2>&1
