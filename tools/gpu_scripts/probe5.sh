python bench.py --force-multi --workload rmat28 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/p5.json 2>gpurun_out/p5.err
python -c "
import json; r=json.load(open('gpurun_out/p5.json'))
print(r['ms_per_step'], json.dumps(r['merge']))"
tail -3 gpurun_out/p5.err
