timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -2
for H in 1 0; do
for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1 grid:4096x4096 rmatx:scale=20,ef=16,seed=1; do
  echo "half=$H $S $(HCC_SUM_HALF=$H python tools/probe.py $S --reps 10 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean'], end=' :: '); continue
    print(round(d['hook_ms'],4), d['hook_kernel'][7:], end=' | ')
")"
done
echo "half=$H adaptive $(HCC_SUM_HALF=$H python tools/probe.py rmatx:scale=24,ef=16,seed=1 --algo adaptive --reps 10 | cut -c60-110)"
done
