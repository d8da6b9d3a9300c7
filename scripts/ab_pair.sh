python -m pytest tests/test_parity_gpu.py tests/test_synth_gpu.py -x -q 2>&1 | tail -3
for i in 1 2; do for k in resident auto; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --kernel $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$k', round(d['value']/1e12,4), 'e2e', round(d['e2e']['value']/1e12,4), 'kern_ms', round(d['roofline']['kernel_ms'],4), d['ambiguous_draws'])"
done; done
python scripts/imbalance.py
