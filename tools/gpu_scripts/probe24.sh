timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
tl() { python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], d.get('exact',''), end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
"; }
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=16,ef=16,seed=1 rmatx:scale=26,ef=16,seed=1 rmatx:scale=28,ef=16,seed=1; do
  R=10; case $S in *28*) R=3;; esac
  echo "$S $(python tools/probe.py $S --reps $R --timeline | tl)"
done
