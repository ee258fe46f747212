timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-e2e --no-classical --no-variants > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('unsharded', round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in r['phase_ms_per_step'].items()})"
python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
import mf_inputs, paper_2312_12732_b200 as mf
n = 16384
A, B = mf_inputs.device_pair("uniform", n, 0)
C = torch.empty_like(A)
for N in (2, 8):
    with mf.Plan(mf.triples.STRASSEN_WINOGRAD, 2, n, shard_rank=0, shard_count=N, profile=True) as p:
        for _ in range(2): p.dgemm(A, B, C)
        torch.cuda.synchronize(); p.profile_read()
        for _ in range(3): p.dgemm(A, B, C)
        ph = p.profile_read()
        print("shard 0 of", N, {k: round(v / ph["calls"], 3) for k, v in ph.items() if k != "calls"})
PY
