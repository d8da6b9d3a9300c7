#!/bin/bash
# Interleaved A/B of library variants (ab/<name>.so, "cur" = in-tree build) on the C1 bench:
#   VARIANTS="noopt pfonly cur" N=2 bash scripts/ab_variants.sh
N=${N:-2}
for i in $(seq $N); do
  for v in $VARIANTS; do
    if [ $v = cur ]; then unset EBL_LIB; else export EBL_LIB=$PWD/ab/$v.so; fi
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['value']/1e12,4), 'e2e', round(d['e2e']['value']/1e12,4), 'kern_ms', round(d['roofline']['kernel_ms'],4), 'amb', d['ambiguous_draws'], 'fb', d['fp64_fallback_draws'])"
  done
done
