"""Phase trace of the small-problem kernel (config 1) from a diagnostic build:
    mkdir -p ab_trace/paper_2312_12732_b200; cp paper_2312_12732_b200/{__init__,triples}.py ab_trace/paper_2312_12732_b200/
    nvcc ... -DMF_TINY_TRACE -c paper_2312_12732_b200/csrc/mf_tiny.cu -o ab_trace/tiny_trace.o   (flags as tools/build_mf.py)
    nvcc ... -shared -cudart static -o ab_trace/paper_2312_12732_b200/libmf.so <other _build objs> ab_trace/tiny_trace.o
    cp tools/tiny_trace.py ab_trace/ && python ab_trace/tiny_trace.py
Results: profiles/tiny_trace_r02.json."""
import ctypes, os, sys
here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, here); sys.path.insert(1, os.path.dirname(here))
import numpy as np, torch, mf_inputs
import paper_2312_12732_b200 as mf
assert mf.LIB_PATH.startswith(here), mf.LIB_PATH
from paper_2312_12732_b200 import triples
n = 64
A, B = mf_inputs.device_pair("uniform", n, 0)
C = torch.empty_like(A)
lib = ctypes.CDLL(mf.LIB_PATH)
with mf.Plan(triples.get("strassen-winograd"), 1, n) as p:
    for _ in range(50):
        p.dgemm(A, B, C)
    torch.cuda.synchronize()
    buf = np.zeros((8, 12), dtype=np.uint64)
    assert lib.mf_debug_tiny_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t0 = buf[:, 0].min()
names = ["start", "A,B,coef staged", "K4 of first product", "products done", "cluster sync 1", "gather done", "cluster sync 2", "C stored"]
for c in range(7):
    print(c, [int(buf[c, i] - t0) for i in range(8)])
print(names)
