cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in cur nofast cur nofast; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python scripts/c1_tail.py $v
done > gpurun_out/ab2.log 2>&1
unset EBL_LIB
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_r02b.log 2>&1
