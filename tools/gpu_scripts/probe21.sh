tl() { python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact',''), end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
"; }
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=20,ef=16,seed=1 rmatx:scale=22,ef=16,seed=1; do
for CFG in "HCC_SUMD=0" "HCC_SUMD=1" "HCC_SUMD=2" "HCC_SUMD=1 HCC_SUM_VOTE=0" "HCC_SUMD=2 HCC_SUM_VOTE=0"; do
  echo "$S $CFG: $(env $CFG python tools/probe.py $S --reps 10 --timeline --check | tl)"
done
done
