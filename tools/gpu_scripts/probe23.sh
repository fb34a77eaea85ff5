S=rmatx:scale=28,ef=16,seed=1
echo "28 default $(python tools/probe.py $S --reps 3 | cut -c60-120)"
echo "28 prefix $(HCC_S0F_PREFIX=1 python tools/probe.py $S --reps 3 --check --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact',''), end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
")"
echo "26 default $(python tools/probe.py rmatx:scale=26,ef=16,seed=1 --reps 3 --check | cut -c60-120)"
echo "26 prefix $(HCC_S0F_PREFIX=1 python tools/probe.py rmatx:scale=26,ef=16,seed=1 --reps 3 --check | cut -c60-120)"
echo "25 prefix exact $(HCC_S0F_PREFIX=1 python tools/probe.py rmatx:scale=25,ef=4,seed=3 --reps 1 --check | grep -o '\"exact\": [a-z]*')"
echo "er26 prefix exact $(HCC_S0F_PREFIX=1 python tools/probe.py erx:n=67108869,m=134217728,seed=3 --reps 1 --check | grep -o '\"exact\": [a-z]*')"
