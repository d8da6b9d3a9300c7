# e2e of the host-buffer pipeline vs chunk count (default zero-copy split: the later half)
for i in 1 2; do
  for c in 2 3 4 5 6 8; do
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chunks $c', 'e2e', round(d['e2e']['value']/1e12,4))"
  done
  for z in 1 3; do
    EBL_PIPE_ZC=$z python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline 6 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chunks 6 zc $z', 'e2e', round(d['e2e']['value']/1e12,4))"
  done
done
