for S in erx:n=16777216,m=268435456,seed=1 rmatx:scale=24,ef=16,seed=1 grid:4096x4096 erx:n=4194304,m=16777216,seed=1; do
  for V in "" "HCC_HOOK_BOTH=1" "" "HCC_HOOK_BOTH=1"; do
    echo "$S [$V] $(env $V python tools/probe.py $S --reps 15 | cut -c60-120)"
  done
  HCC_HOOK_BOTH=1 python tools/probe.py $S --reps 3 --check --timeline > gpurun_out/p77.log 2>&1; echo "  $(head -1 gpurun_out/p77.log | grep -o 'exact[^,}]*')"
  python - <<'PY'
import json
L=open('gpurun_out/p77.log').read().strip().splitlines()
rows=[json.loads(l) for l in L if '"hook_kernel"' in l][-5:]
print('   ', [(d['hook_kernel'][7:], round(d['hook_ms'],3), round(d['compress_ms'],3)) for d in rows])
PY
done
