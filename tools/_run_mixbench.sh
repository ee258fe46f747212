timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -2
for bn in 128 64; do MF_LEAF_BN=$bn timeout 300 python bench.py --config c2-sw1-4096 --steps 20 --no-cpu --no-e2e > gpurun_out/b4096_$bn.json 2>gpurun_out/b4096_$bn.err; python -c "
import json; d=json.load(open('gpurun_out/b4096_$bn.json')); r=d['roofline']
print('bn=$bn', round(d['value'],3), round(d['ms_per_step'],4), round(r['achieved'],3), round(r['frac'],4), d['speedup_vs_cublas'], {k: round(v,3) for k,v in r['phase_ms_per_step'].items()})"; done
for bn in 64; do MF_LEAF_BN=$bn timeout 300 python bench.py --no-cpu --no-e2e --no-classical > gpurun_out/b16k_$bn.json 2>gpurun_out/b16k_$bn.err; python -c "
import json; d=json.load(open('gpurun_out/b16k_$bn.json')); r=d['roofline']
print('16k bn=$bn', round(d['value'],3), round(d['ms_per_step'],4), round(r['achieved'],3), round(r['frac'],4))"; done
