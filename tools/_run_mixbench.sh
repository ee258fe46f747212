timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -2
for k in 0 1; do MF_LEAF_PERSIST=$k timeout 300 python bench.py --no-cpu --no-e2e --no-classical > gpurun_out/b_p$k.json 2>gpurun_out/b_p$k.err; python -c "
import json; d=json.load(open('gpurun_out/b_p$k.json')); r=d['roofline']
print('persist=$k', round(d['value'],3), round(d['ms_per_step'],3), round(r['achieved'],3), round(r['frac'],4), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()}, d['variants'][0]['value'])"; done
for k in 0 1; do MF_LEAF_PERSIST=$k timeout 300 python bench.py --config c2-sw1-4096 --steps 20 --no-cpu --no-e2e --no-classical --no-variants > gpurun_out/b4_p$k.json 2>gpurun_out/b4_p$k.err; python -c "
import json; d=json.load(open('gpurun_out/b4_p$k.json')); r=d['roofline']
print('4096 persist=$k', round(d['value'],3), round(r['frac'],4))"; done
