for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1; do
  for V in "HCC_BOTH_LAST=0" "HCC_BOTH_LAST=1"; do
    env $V python tools/probe.py $S --reps 5 --timeline > gpurun_out/p87.log 2>&1
    echo "$S [$V] $(head -1 gpurun_out/p87.log | cut -c60-110)"
    python - <<'PY'
import json
L=open('gpurun_out/p87.log').read().strip().splitlines()
rows=[json.loads(l) for l in L if '"hook_kernel"' in l][-5:]
print('   ', [(d['hook_kernel'][7:], d['edges_in']>>20, round(d['hook_start_ms'],3), round(d['hook_ms'],3), round(d['compress_ms'],3), round(d['compress_end_ms'],3)) for d in rows])
PY
  done
done
