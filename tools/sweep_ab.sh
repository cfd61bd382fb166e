# usage: bash tools/sweep_ab.sh libs...  -- sweep + step-config timings per build
for L in "$@"; do
  PSWE_LIB_PATH=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$L', round(d['ms_per_step'],3), ' '.join(f\"{p['n']}/{p['M']}:{p['ms']*1e3:.0f}\" for p in d['sweep']), ' '.join(f\"{s['config']}:{s.get('ms_per_step',0)*1e3:.0f}\" for s in d['step_configs']))"
done
