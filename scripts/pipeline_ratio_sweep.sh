# e2e of the host-buffer pipeline vs chunk count and geometric chunk ratio (EBL_PIPE_RATIO; > 1: later chunks larger)
for i in 1 2; do
  for r in 1.0 1.2 1.5 2.0; do
    for c in 4 6; do
      EBL_PIPE_RATIO=$r python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pipeline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ratio $r chunks $c', 'e2e', round(d['e2e']['value']/1e12,4))"
    done
  done
done
