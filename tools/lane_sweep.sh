# Chunk/lane policy A/B at the small-M points: sweep timings per (PSWE_MINPH, PSWE_MINMB)
for cfg in "16 24" "8 24" "4 24" "4 48" "2 24" "8 96" "4 96"; do
  set -- $cfg
  PSWE_MINPH=$1 PSWE_MINMB=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-steps 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('minph=$1 minmb=$2', ' '.join('%d/%d:%.1f' % (s['n'], s['M'], 1e3*s['ms']) for s in d['sweep']))"
done
