# small-size sweep timings per build: bash tools/sweep_ab2.sh libA.so libB.so
for L in "$@" "$@"; do
  echo -n "$(basename $L) "; PSWE_LIB_PATH=$L timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print(' '.join('%d/%d:%.1f' % (s['n'], s['M'], 1e3*s['ms']) for s in d['sweep'] if s['n'] <= 256), '|', ' '.join('%s:%.1f' % (s['config'], 1e3*s.get('ms_per_step', 0)) for s in d['step_configs'][:4]))"
done
