for S in rmatx:scale=24,ef=16,seed=1 rmatx:scale=28,ef=16,seed=1; do
echo "$S plain $(python tools/probe.py $S --reps 5 | cut -c60-150)"
echo "$S sumd  $(HCC_SUMD=1 python tools/probe.py $S --reps 5 --check --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact')); continue
    print(round(d['hook_ms'],4), d['hook_kernel'], end=' | ')
")"
done
echo "er sumd $(HCC_SUMD=1 python tools/probe.py erx:n=16777216,m=268435456,seed=1 --reps 5 --check | cut -c60-150)"
