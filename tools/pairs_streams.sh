# config-4 sweep: pairs/s for a batch of 64 256^3 pairs at several in-flight counts (one GPU)
for k in 4 8 12; do  # ~4 min per run (host-side input generation)
  python bench.py --steps 3 --warmup 3 --cpu-budget 0 --pairs 64 --streams $k 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d['full_registration']['batch']; print('streams', $k, 'pairs/s', round(b['pairs_per_s'],1))"
done
