#!/bin/bash
# A/B timing of the in-tree library against ab/libember_b200_prev.so on the same box,
# interleaved: python bench.py ... under each, N rounds.
N=${N:-3}
for i in $(seq $N); do
  for v in prev cur; do
    if [ $v = prev ]; then export EBL_LIB=$PWD/ab/libember_b200_prev.so; else unset EBL_LIB; fi
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['value']/1e12,4), 'e2e', round(d['e2e']['value']/1e12,4), 'kern_ms', round(d['roofline']['kernel_ms'],4))"
  done
done
