timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "host" 2>&1 | tail -2
for c in c3-sw2-16384 c2-sw1-4096 c4b-sw2-13824 c4a-ld1-13824; do timeout 300 python bench.py --config $c --no-cpu --no-classical > gpurun_out/b_e2e_$c.json 2>gpurun_out/b_e2e_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_e2e_$c.json'))
print('$c', round(d['value'],3), round(d['e2e']['value'],3), round(d['e2e']['ms_per_step'],2))"; done
