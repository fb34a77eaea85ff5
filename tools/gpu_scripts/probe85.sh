for S in rmatx:scale=24,ef=16,seed=1 erx:n=16777216,m=268435456,seed=1; do
  for L in "" "HCC_LIB=paper_1612_01178_b200/lib/variants/ept4.so" "HCC_LIB=paper_1612_01178_b200/lib/variants/ept16.so"; do
    python tools/probe.py $S --reps 15 --timeline > gpurun_out/p85.log 2>&1 || true
    echo "$S [$L] $(env $L python tools/probe.py $S --reps 20 | cut -c60-120)"
    env $L python tools/probe.py $S --reps 5 --timeline > gpurun_out/p85.log 2>&1
    python - <<'PY'
import json
L=open('gpurun_out/p85.log').read().strip().splitlines()
rows=[json.loads(l) for l in L if '"hook_kernel"' in l][-5:]
print('   ', [(d['hook_kernel'][7:], round(d['hook_ms'],3), round(d['compress_ms'],3)) for d in rows])
PY
  done
done
