for S in erx:n=16777217,m=268435456,seed=2 erx:n=67108864,m=268435456,seed=3 erx:n=67108864,m=1073741824,seed=3 rmatx:scale=26,ef=16,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 5 --timeline --check | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact'), end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
")"
done
