# one A/B sample for tools/ab_so.sh: fused kernel and whole-evaluation time at 256^3 (config 3)
python bench.py --steps 50 --warmup 5 --no-register --cpu-budget 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 kernel_ms', round(d['roofline']['kernel_ms'],4), 'ms_per_step', round(d['ms_per_step'],4))"
