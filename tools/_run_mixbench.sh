timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -2
for bm in 0 2; do MF_LEAF_BMODE=$bm timeout 300 python bench.py --no-e2e --no-cpu --no-classical > gpurun_out/bench_bm$bm.json 2>gpurun_out/bench_bm$bm.err; python -c "
import json; d=json.load(open('gpurun_out/bench_bm$bm.json')); r=d['roofline']
print('bmode=$bm', round(d['value'],3), round(d['ms_per_step'],3), round(r['achieved'],3), round(r['frac'],4), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()})"; done
