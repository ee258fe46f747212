timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -3
for L in 3; do timeout 300 python bench.py --levels $L --no-cpu --no-e2e > gpurun_out/b_L$L.json 2>gpurun_out/b_L$L.err; tail -2 gpurun_out/b_L$L.err; python -c "
import json; d=json.load(open('gpurun_out/b_L$L.json')); r=d['roofline']
print('L=$L', round(d['value'],3), round(d['ms_per_step'],4), round(r['achieved'],3), round(r['frac'],4), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()}, d['max_scaled_error'], d.get('speedup_vs_cublas'))"; done
timeout 300 python bench.py --triple laderman --n 13824 --levels 2 --no-cpu --no-e2e > gpurun_out/b_ld2.json 2>gpurun_out/b_ld2.err; tail -2 gpurun_out/b_ld2.err; python -c "
import json; d=json.load(open('gpurun_out/b_ld2.json')); r=d['roofline']
print('LD2', round(d['value'],3), round(d['ms_per_step'],4), round(r['achieved'],3), round(r['frac'],4), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()}, d['max_scaled_error'], d.get('speedup_vs_cublas'))"
