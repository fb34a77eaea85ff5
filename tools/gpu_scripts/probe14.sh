S=rmatx:scale=28,ef=16,seed=1
for PAD in 0x100000 0x2000000; do
echo "== pad $PAD"
HCC_S0B_PAD=$PAD python tools/probe.py $S --reps 3 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean']); continue
    print({k:d[k] for k in ('hook_ms','compress_ms','hook_start_ms','hook_end_ms','compress_start_ms','compress_end_ms','hook_kernel')})
"
done
