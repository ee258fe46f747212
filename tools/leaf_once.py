"""Two mf_dgemm calls of one configuration (for ncu captures of the second
call's kernels).  python tools/leaf_once.py [n] [levels] [fuse_postadd]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402
from paper_2312_12732_b200 import triples  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
fuse = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A, B = mf_inputs.device_pair("uniform", n, 0)
with mf.Plan(triples.get("strassen-winograd"), L, n, fuse_postadd=fuse) as p:
    for _ in range(2):
        C = p.dgemm(A, B)
    torch.cuda.synchronize()
print("ok", n, L, fuse, float(C[0, 0]))
