S=rmatx:scale=28,ef=16,seed=1
R=0,536870912
python tools/probe.py $S --range $R --reps 3 --timeline | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln)
    if 'spec' in d: print(d['ms_mean']); continue
    print({k:d[k] for k in ('hook_ms','compress_ms','edges_in','edges_out','hook_start_ms','compress_end_ms','hook_kernel')})
"
for PL in adapt:7:4 adapt:7:3 adapt:6:3 adapt:5:3 adapt:5:2 adapt:4:2 adapt:3:2 adapt:2:2 adapt:1:2; do
echo "$PL $(HCC_PLAN=$PL python tools/probe.py $S --range $R --reps 3 | cut -c60-100)"
done
for NS in 2 3 4; do
echo "nshift $NS $(HCC_PLAN_NSHIFT=$NS python tools/probe.py $S --range $R --reps 3 | cut -c60-100)"
done
R=0,1073741824
for PL in adapt:7:4 adapt:5:3 adapt:4:2 adapt:3:2; do
echo "N4 $PL $(HCC_PLAN=$PL python tools/probe.py $S --range $R --reps 3 | cut -c60-100)"
done
