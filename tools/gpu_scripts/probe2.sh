python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-adaptive --rmat28-e2e-steps 0 > gpurun_out/p2_bench.json 2>gpurun_out/p2_bench.err
python -c "
import json; d=json.load(open('gpurun_out/p2_bench.json'))
print(d['ms_per_step']); r=d['rmat28']; print(r['ms_per_step'], json.dumps(r['merge']))"
python tools/probe.py rmatx:scale=28,ef=16,seed=1 --reps 3 --forest --timeline
