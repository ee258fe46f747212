import os, sys
sys.path.insert(0, "/root/repo")
os.environ["MF_LEAF_SPLIT"] = "1"
import torch, mf_inputs
import paper_2312_12732_b200 as mf
from paper_2312_12732_b200 import triples
n = int(sys.argv[1]); t = triples.get("strassen-winograd")
A, B = mf_inputs.device_pair("uniform", n, 0)
with mf.Plan(t, 2, n) as p:
    ref = p.dgemm(A, B).clone()
os.environ.setdefault("MF_LEAF_2CTA", "1")
for trial in range(3):
    with mf.Plan(t, 2, n, fuse_postadd=1) as p:
        C1 = p.dgemm(A, B).clone()
        C2 = p.dgemm(A, B).clone()
    torch.cuda.synchronize()
    print("fresh plan: launch1 mism", int((C1 != ref).sum()), "launch2 mism", int((C2 != ref).sum()))
