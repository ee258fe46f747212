"""n=64 SW^1 (config 1): per-call time of mf_dgemm (eager and graph) vs cuBLAS,
CUDA events over 200 back-to-back calls.  python tools/tiny_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mf_inputs
import paper_2312_12732_b200 as mf
from paper_2312_12732_b200 import triples
n = 64
A, B = mf_inputs.device_pair("uniform", n, 0)
C = torch.empty_like(A)
st = torch.cuda.Stream()
def t(fn, reps=200):
    with torch.cuda.stream(st):
        for _ in range(20): fn()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps): fn()
        e1.record(st)
        st.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
res = {"cublas_us": t(lambda: torch.matmul(A, B, out=C))}
with mf.Plan(triples.get("strassen-winograd"), 1, n) as p:
    res["mf_eager_us"] = t(lambda: p.dgemm(A, B, C, stream=st))
with mf.Plan(triples.get("strassen-winograd"), 1, n, graph=True) as p:
    res["mf_graph_us"] = t(lambda: p.dgemm(A, B, C, stream=st))
print(os.environ.get("MF_TINY_CS", "default"), {k: round(v, 2) for k, v in res.items()})
