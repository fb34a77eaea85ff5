timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest8.log
tail -2 gpurun_out/r2_gputest8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "rmat24 $(python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 20 | cut -c60-120)"
