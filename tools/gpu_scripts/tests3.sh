timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest3.log
tail -3 gpurun_out/r2_gputest3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
