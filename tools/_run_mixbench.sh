timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-classical > gpurun_out/b_$i.json 2>gpurun_out/b_$i.err; python -c "
import json; d=json.load(open('gpurun_out/b_$i.json')); r=d['roofline']
print('run$i', round(d['value'],3), round(d['ms_per_step'],4), round(r['achieved'],3), round(r['frac'],4), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()})"; done
