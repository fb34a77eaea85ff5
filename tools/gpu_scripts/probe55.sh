timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for S in rmatx:scale=16,ef=16,seed=1 rmatx:scale=18,ef=16,seed=1 grid:512x512 rmatx:scale=20,ef=16,seed=1 rmatx:scale=24,ef=16,seed=1; do
  echo "$S $(python tools/probe.py $S --reps 20 | cut -c60-120)"
done
timeout 600 python bench.py --workload rmat16 --no-rmat28 --no-adaptive --e2e-steps 2 > gpurun_out/r2_bench_v6_rmat16.json 2>/dev/null; echo "rmat16 rc=$?"
