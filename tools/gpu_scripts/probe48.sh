for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096; do
  for M in 2 8 32; do
    HCC_SMALL_MULT=$M python tools/probe.py $S --reps 10 --timeline > gpurun_out/p48.log 2>&1
    echo "$S mult=$M $(head -1 gpurun_out/p48.log | cut -c60-110)"
    python - <<'PY'
import json
L=open('gpurun_out/p48.log').read().strip().splitlines()
rows=[json.loads(l) for l in L if '"hook_kernel"' in l][-5:]
print('   ', [(d['hook_kernel'][7:], round(d['hook_ms'],3), round(d['compress_ms'],3)) for d in rows])
PY
  done
done
