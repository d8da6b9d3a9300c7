#!/bin/bash
# A/B of library variants on the other BASELINE configs (scripts/bench_configs.py):
#   VARIANTS="prev cur" CONFIGS=c2,c3 bash scripts/ab_configs.sh
for v in $VARIANTS; do
  if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
  python scripts/bench_configs.py --configs ${CONFIGS:-c2} --iters ${ITERS:-3} 2>/dev/null | \
    python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', d['config'][:3], '%.4g'%d['value'], d['unit'], 'ms', round(d['ms_per_step'],3))"
done
