# e2e of the host-buffer pipeline vs how many trailing chunks write their output zero-copy (EBL_PIPE_ZC)
for i in 1 2; do
  for z in 1 2 4; do
    for c in 4 8; do
      EBL_PIPE_ZC=$z python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('zc $z chunks $c', 'e2e', round(d['e2e']['value']/1e12,4))"
    done
  done
done
